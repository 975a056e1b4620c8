# end-of-session GPU pass: smoke, GPU suite, C3 bench, C3 bench launch list, per-solve kernel tables,
# ncu --set full of C3's coarse dataflow kernel
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02i_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02i_pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/r02i_bench_C3.json 2> gpurun_out/r02i_bench_C3.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C3 C5; do
  timeout 400 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/r02i_solve_$c.csv python tools/prof_solve.py $c > gpurun_out/r02i_solve_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r02i_c3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_coarse_dataflow --launch-skip 2 -c 1 -o gpurun_out/r02i_df_full_C3 -f python tools/prof_solve.py C3 > gpurun_out/r02i_ncu_fulldf.log 2>&1
tail -2 gpurun_out/r02i_pytest_gpu.log; tail -1 gpurun_out/r02i_smoke.log
