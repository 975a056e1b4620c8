python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric_gauss or sparse or pcg_parity or apply" 2>&1 | tail -3
for cfg in C3 C4 C2; do for sy in 0 1; do
DDG_GJ_SYM=$sy timeout 300 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/gjsym_${cfg}_$sy.json 2> gpurun_out/gjsym_${cfg}_$sy.err
python -c "import json;d=json.load(open('gpurun_out/gjsym_${cfg}_$sy.json'));print('$cfg sym=$sy setup', d['config']['t_setup_s'], 'solve', round(d['ms_per_step'],2), d['config']['iterations'])" 2>&1 | tail -1
done; done
