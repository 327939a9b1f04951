timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_gputests_final.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_gputests_final.log
bash tools/capture_profiles.sh all > gpurun_out/r2_capture.log 2>&1; echo capture rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err; echo ref rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
