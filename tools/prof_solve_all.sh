M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C2 C5; do
timeout 300 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/solve_$c.csv python tools/prof_solve.py $c > gpurun_out/solve_$c.log 2>&1; echo "$c rc=$?"
done
