# full ncu capture of one colour-sweep SYMV launch (ring and classic) on C2
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_ring --launch-skip 3 -c 1 -o gpurun_out/ring_c2 -f python tools/prof_solve.py C2 > gpurun_out/ncu_ring.log 2>&1
echo "ring rc=$?"
DDG_SYMV=classic ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_symv\(" --launch-skip 3 -c 1 -o gpurun_out/classic_c2 -f python tools/prof_solve.py C2 > gpurun_out/ncu_classic.log 2>&1
echo "classic rc=$?"
