# round-2 GPU pass: tests, bench lines for every config, per-solve kernel lists,
# the C3 bench launch list, full captures of the dominant kernels (C3, C5)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench rc=$?"
for c in ${CFGS:-C5 C2 C4 C1}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in ${SOLVE_CFGS:-C3 C5 C2 C4}; do
  timeout 400 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/solve_$c.csv python tools/prof_solve.py $c > gpurun_out/solve_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches_C3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_whole --launch-skip 5 -c 1 -o gpurun_out/whole_full_C3 -f python tools/prof_solve.py C3 > gpurun_out/ncu_full3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring2 --launch-skip 5 -c 1 -o gpurun_out/ring2_full_C5 -f python tools/prof_solve.py C5 > gpurun_out/ncu_full5.log 2>&1
echo done
