set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_three_level.py -x -q 2>&1 | tail -15
for cfg in "C2 2" "C3 4" "C5 4" "C4 2"; do set -- $cfg; timeout 600 python bench.py --config $1 --levels 3 --factor $2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b3_$1.json 2> gpurun_out/b3_$1.err; echo "$1 exit $?"; tail -c 600 gpurun_out/b3_$1.err; done
