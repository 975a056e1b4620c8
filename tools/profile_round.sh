# round profile: bench lines for every config, per-solve launch lists, C2 bench launch list,
# full ncu captures of k_symv_ring (C2), k_symv_ring2 (C3), k_coarse_dataflow (C2), k_gjb_gemm (C4 setup)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_round.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C3 C5 C4 C1; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C2 C3 C5 C4; do
  timeout 400 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/solve_$c.csv python tools/prof_solve.py $c > gpurun_out/solve_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring --launch-skip 5 -c 1 -o gpurun_out/ring_full_C2 -f python tools/prof_solve.py C2 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring2 --launch-skip 5 -c 1 -o gpurun_out/ring2_full_C3 -f python tools/prof_solve.py C3 > gpurun_out/ncu_full3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_coarse_dataflow --launch-skip 2 -c 1 -o gpurun_out/df_full_C2 -f python tools/prof_solve.py C2 > gpurun_out/ncu_fulldf.log 2>&1
