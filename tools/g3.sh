python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitions.py -x -q > gpurun_out/pytest_band.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_band.log
for v in "" "DDG_BAND_TILES=6" "DDG_BAND_TILES=4" "DDG_BAND=0"; do
  for c in C3 C5; do env $v timeout 300 python tools/symv_probe.py $c 3 2>&1 | tail -1; done
done
