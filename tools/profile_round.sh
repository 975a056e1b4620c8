# round profile: bench lines for every config, per-kernel launch lists of one solve (C2, C3, C5, C4),
# the C2 bench launch list, one full ncu capture of k_symv_ring
set -x
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C3 C5 C4 C1; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C2 C3 C5 C4; do
  timeout 400 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/solve_$c.csv python tools/prof_solve.py $c > gpurun_out/solve_$c.log 2>&1
done
if [ -n "$FULL" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring --launch-skip 5 -c 1 -o gpurun_out/ring_full_C2 -f python tools/prof_solve.py C2 > gpurun_out/ncu_full.log 2>&1
fi
