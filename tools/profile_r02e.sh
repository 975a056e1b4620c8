# round-2 final GPU pass: tests, smoke, bench lines for every config, per-solve
# kernel lists, the C3 bench launch list
set -x
T=${T:-e}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${T}.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${T}.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${T}_C3.json 2> gpurun_out/bench_${T}_C3.err; echo "bench rc=$?"
for c in C5 C2 C4 C1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_${T}_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C3 C5 C2 C4; do
  timeout 400 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/solve_${T}_$c.csv python tools/prof_solve.py $c > gpurun_out/solve_${T}_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches_${T}_C3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${T}.log 2>&1
echo done
if [ -n "$RING2_CAPTURE" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring2 --launch-skip 5 -c 1 -o gpurun_out/ring2_full_C5_${T} -f python tools/prof_solve.py C5 > gpurun_out/ncu_ring2_${T}.log 2>&1
fi
if [ -n "$CHOL_BENCH" ]; then
  for c in C2 C4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --local-variant cholesky > gpurun_out/bench_${T}_chol_$c.json 2> gpurun_out/bench_${T}_chol_$c.err; done
fi
