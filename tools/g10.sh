python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
DDG_DEBUG_FILL=255 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_partitions.py -q -x 2>&1 | tail -5
timeout 1500 python -m pytest tests/test_gpu_full_parity.py tests/test_gpu_loopback.py -q 2>&1 | tail -5
