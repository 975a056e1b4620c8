python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in C2 C5; do for leaf in 256 512 1024 2048 4096; do
DDG_ND_LEAF=$leaf timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/leaf_${cfg}_$leaf.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/leaf_${cfg}_$leaf.json'));print('$cfg leaf=$leaf', round(d['ms_per_step'],3), round(d['kernel_ms_per_solve']['coarse'],3), d['config']['coarse_solve_bytes']/1e9)"
done; done
