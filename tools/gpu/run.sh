# scratch command file for gpurun calls; the last one: the full GPU suite, the default bench line and smoke()
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_c4_final.json 2> gpurun_out/bench_c4_final.err; echo bench rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
