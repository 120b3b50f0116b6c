#!/bin/bash
# Round-2 GPU round trip: build, all GPU tests, bench lines for every config,
# the balanced-router line and a 2-rank (gloo, shared GPU) run of bench.py.
set -u
mkdir -p gpurun_out
python -m paper_2306_06446_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2 c3 c4 c5}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench_$c.log 2>&1
  head -c 400 gpurun_out/bench_$c.log; echo
done
timeout 600 python bench.py --router balanced --steps 10 --warmup 3 --skip-cpu > gpurun_out/bench_c2_balanced.log 2>&1
head -c 300 gpurun_out/bench_c2_balanced.log; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --skip-cpu --skip-kernels \
  > gpurun_out/bench_2rank.log 2>&1
head -c 300 gpurun_out/bench_2rank.log; echo
