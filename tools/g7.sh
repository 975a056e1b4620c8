python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in "DDG_WHOLE_PLAN=0" "DDG_WHOLE_PLAN=1"; do
  env $v timeout 300 python tools/symv_probe.py C3 3 2>&1 | tail -1
  env $v DDG_RING_MIN_MB=0 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pcg_parity" 2>&1 | tail -1
done
