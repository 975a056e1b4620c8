python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_three_level.py -x -q 2>&1 | tail -2
for cfg in C3 C4 C5 C2; do for fl in 0 1; do
DDG_FLAT_COARSE=$fl timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/flat_${cfg}_$fl.json 2> gpurun_out/flat_${cfg}_$fl.err
python -c "import json;d=json.load(open('gpurun_out/flat_${cfg}_$fl.json'));print('$cfg flat=$fl', round(d['ms_per_step'],3), round(d['kernel_ms_per_solve']['coarse'],3))" 2>&1 | tail -1
done; done
