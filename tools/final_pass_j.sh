# last GPU pass of round 2 (r02j): smoke, GPU suite, bench lines of all five configs and the
# reference arm at HEAD, ncu --set full of the dominant kernel of C3 (k_symv_whole) and C5 (k_symv_ring2)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02j_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02j_pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/r02j_bench_C3.json 2> gpurun_out/r02j_bench_C3.err
for c in C5 C2 C4 C1; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02j_bench_$c.json 2> gpurun_out/r02j_bench_$c.err
done
timeout 400 python bench.py --impl reference > gpurun_out/r02j_bench_reference.json 2> gpurun_out/r02j_bench_reference.err
timeout 400 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_whole --launch-skip 5 -c 1 -o gpurun_out/r02j_whole_C3 -f python tools/prof_solve.py C3 > gpurun_out/r02j_ncu_whole_C3.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring2 --launch-skip 5 -c 1 -o gpurun_out/r02j_ring2_C5 -f python tools/prof_solve.py C5 > gpurun_out/r02j_ncu_ring2_C5.log 2>&1
for f in r02j_whole_C3 r02j_ring2_C5; do
  ncu -i gpurun_out/$f.ncu-rep --page details > gpurun_out/${f}_details.txt 2>&1
done
tail -2 gpurun_out/r02j_pytest_gpu.log; tail -1 gpurun_out/r02j_smoke.log; cat gpurun_out/r02j_bench_C3.json | cut -c1-400
