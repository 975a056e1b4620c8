python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_loopback.py -q 2>&1 | tail -4; done
DDG_WHOLE_PLAN=1 timeout 600 python -m pytest tests/test_gpu_loopback.py -q 2>&1 | tail -4
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_loopback.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
