python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fr.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ring or parity or bitwise" 2>&1 | tail -3
for cfg in C2 C4; do for fr in 0 1; do
DDG_RING_FUSED_RED=$fr timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fr_${cfg}_$fr.json 2> gpurun_out/fr_${cfg}_$fr.err
python -c "import json;d=json.load(open('gpurun_out/fr_${cfg}_$fr.json'));print('$cfg fr=$fr', round(d['ms_per_step'],3), d['config']['iterations'], {k:round(v,2) for k,v in d['kernel_ms_per_solve'].items()}, round(d['roofline']['frac'],3))"
done; done
