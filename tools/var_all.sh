# parity tests, then kernel variants per config (short timeouts: a hang costs GPU budget)
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in ${CONFIGS:-C2 C3 C5 C4 C1}; do
  timeout 300 python tools/variants.py $c "" ${VARIANTS:-"DDG_SYMV=classic"} > gpurun_out/var_$c.log 2>&1; echo "$c rc=$?"
done
