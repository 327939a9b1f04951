for lib in build/ab/base.so build/ab/ib.so; do
  echo "== $lib"
  RASTERBOUND_B200_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__sass_inst_executed_op_shared_atom.sum --clock-control none -k regex:k_point_pass_ring -c 4 python tools/ablate.py 1e8 2>&1 | grep -E "k_point_pass_ring|duration|inst_executed|bank|atom" | head -30
done
