python tools/fp64_peak.py > gpurun_out/fp64_peak.json 2>&1
timeout 300 python tools/setup_profile.py C3 > gpurun_out/setup_prof4_C3.md 2>&1
timeout 300 python tools/setup_profile.py C4 > gpurun_out/setup_prof4_C4.md 2>&1
DDG_GJ_PIPE=0 timeout 300 python tools/setup_profile.py C4 > gpurun_out/setup_prof4_C4_nopipe.md 2>&1
timeout 300 python tools/gjunit.py 97 161 300 > gpurun_out/gjunit4.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_cholesky.py tests/test_gpu_three_level.py -x -q > gpurun_out/gpu_tests4.log 2>&1
timeout 600 python tools/setup_times.py C2 C3 C4 C5 > gpurun_out/setup_times4.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C3 C5; do
  LOCAL_VARIANT=1 timeout 400 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/solve_chol_$c.csv python tools/prof_solve.py $c > gpurun_out/solve_chol_$c.log 2>&1
done
LOCAL_VARIANT=1 timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_chol_solve --launch-skip 5 -c 1 -o gpurun_out/chol_full_C3 -f python tools/prof_solve.py C3 > gpurun_out/ncu_chol3.log 2>&1
LOCAL_VARIANT=1 timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_chol_solve --launch-skip 5 -c 1 -o gpurun_out/chol_full_C5 -f python tools/prof_solve.py C5 > gpurun_out/ncu_chol5.log 2>&1
echo done
