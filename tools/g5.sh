python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitions.py -x -q -k "path or full or pcg_parity" > gpurun_out/pytest_whole.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_whole.log
for v in "" "DDG_RING2_SPLIT=1" "DDG_COMPACT=0" "DDG_RING_NB=3" "DDG_RING_TILES=8"; do
  env $v timeout 300 python tools/symv_probe.py C5 3 2>&1 | tail -1
done
for v in "DDG_RING_WHOLE=0" "DDG_RING_WHOLE=0 DDG_RING2_SPLIT=1"; do
  env $v timeout 300 python tools/symv_probe.py C3 3 2>&1 | tail -1
done
