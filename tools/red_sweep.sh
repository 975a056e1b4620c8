python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for cfg in C2 C4; do
timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/red_${cfg}.json 2> gpurun_out/red_${cfg}.err
python -c "import json;d=json.load(open('gpurun_out/red_${cfg}.json'));print('$cfg', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['kernel_ms_per_solve'].items()})" 2>&1 | tail -1
done
