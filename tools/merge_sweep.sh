python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in 0 3; do DDG_ND_MERGE=$m timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sparse" 2>&1 | tail -1; done
for cfg in C2 C5 C3; do for m in 0 1 2 3 4 6; do
DDG_ND_MERGE=$m timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/merge_${cfg}_$m.json 2> gpurun_out/merge_${cfg}_$m.err
python -c "import json;d=json.load(open('gpurun_out/merge_${cfg}_$m.json'));print('$cfg merge=$m', round(d['ms_per_step'],3), round(d['kernel_ms_per_solve']['coarse'],3), d['config']['coarse_solve_bytes']/1e9, d['config']['t_setup_s'])" 2>&1 | tail -1
done; done
