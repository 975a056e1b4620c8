python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pcg_small -s 2 -c 1 -o gpurun_out/small_C1 -f python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1
