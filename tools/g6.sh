python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python tools/symv_probe.py C5 3 2>&1 | tail -1; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench rc=$?"
for c in C5 C2 C4 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
