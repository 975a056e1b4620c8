python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_whole --launch-skip 5 -c 1 -o gpurun_out/whole2_full_C3 -f python tools/prof_solve.py C3 > gpurun_out/ncu_w.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring2 --launch-skip 5 -c 1 -o gpurun_out/ring2b_full_C5 -f python tools/prof_solve.py C5 > gpurun_out/ncu_r.log 2>&1
