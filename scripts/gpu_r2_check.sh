set -u
mkdir -p gpurun_out
python -m paper_2306_06446_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu > gpurun_out/bench_c2.log 2>&1
head -c 600 gpurun_out/bench_c2.log; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --skip-cpu --skip-kernels > gpurun_out/bench_2rank.log 2>&1
head -c 400 gpurun_out/bench_2rank.log; echo
