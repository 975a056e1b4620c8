python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in "" "DDG_BAND_SLEEP=64" "DDG_BAND_TILES=4" "DDG_BAND_TILES=6"; do
  for c in C3 C5; do env $v timeout 300 python tools/symv_probe.py $c 3 2>&1 | tail -1; done
done
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_symv_band --launch-skip 5 -c 1 -o gpurun_out/band_full_C3 -f python tools/prof_solve.py C3 > gpurun_out/ncu_band3.log 2>&1
