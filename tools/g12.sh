python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
DDG_SMALL_TRACE=1 timeout 120 python tools/small_trace.py > gpurun_out/trace.log 2>&1
grep -i "small\|launch\|iters\|probe\|gaps\|clock" gpurun_out/trace.log
timeout 120 python tools/small_check.py 2>&1 | tail -3
