# r02j, second call: bench.py under the driver's torchrun launch line (1 rank), three-level and Cholesky-variant lines at HEAD
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02j_bench_C3_torchrun.json 2> gpurun_out/r02j_bench_C3_torchrun.err
echo "torchrun rc=$?"
timeout 600 python bench.py --config C3 --levels 3 --factor 2 --steps 10 --warmup 3 > gpurun_out/r02j_bench_3level_C3.json 2> gpurun_out/r02j_bench_3level_C3.err
timeout 600 python bench.py --config C3 --local-variant cholesky --steps 5 --warmup 3 > gpurun_out/r02j_bench_C3_cholesky.json 2> gpurun_out/r02j_bench_C3_cholesky.err
for f in gpurun_out/r02j_bench_C3_torchrun.json gpurun_out/r02j_bench_3level_C3.json gpurun_out/r02j_bench_C3_cholesky.json; do tail -1 $f | cut -c1-260; echo; done
