#!/bin/bash
# quick per-config bench (no CPU baseline); results in gpurun_out/bench_<cfg>.json
for c in ${@:-C2 C5 C3 C4 C1}; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -2 gpurun_out/bench_$c.err
done
