#!/bin/bash
# Round-2 evidence on one GPU: tests, per-op DRAM traffic of one forward,
# the bench's ncu launch list, ncu --set full of the fused MLP kernel at both
# stage shapes, the binary-attention bench, and bench lines for every config.
# Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -m paper_2306_06446_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/traffic.csv \
  python scripts/profile_forward.py --record gpurun_out/op_calls.json > gpurun_out/traffic.log 2>&1
python scripts/ncu_traffic.py gpurun_out/traffic.csv gpurun_out/op_calls.json gpurun_out/ncu_traffic.json \
  > gpurun_out/traffic_summary.txt 2>&1
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json 2>/dev/null
for dd in 32 64; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:mlp_kernel -c 1 \
    --profile-from-start off -o gpurun_out/full_mlp$dd -f python scripts/mlp_one.py $dd \
    > gpurun_out/ncu_full_mlp$dd.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --skip-cpu > gpurun_out/launches_bench.log 2>&1
timeout 600 python scripts/attn_bench.py --debug > gpurun_out/attn_bench.txt 2>&1
timeout 300 python scripts/mlp_bench.py 0 > gpurun_out/mlp_bench.txt 2>&1
MLP_SHAPES="160,640,50176" timeout 300 python scripts/mlp_bench.py 0 r4 r8 >> gpurun_out/mlp_bench.txt 2>&1
QKV_PRODUCT=1 timeout 300 python scripts/qkv_roles.py > gpurun_out/qkv_bench.txt 2>&1
timeout 300 python scripts/qkv_roles.py 0 1 2 34 >> gpurun_out/qkv_bench.txt 2>&1
timeout 300 python scripts/gemm_roles.py 0 >> gpurun_out/qkv_bench.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/fwd_launches.csv python scripts/fwd_launches.py > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/fwd_launches.csv > gpurun_out/fwd_summary.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1
head -c 300 gpurun_out/bench_c2.log; echo
for c in c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --skip-cpu > gpurun_out/bench_$c.log 2>&1
  head -c 200 gpurun_out/bench_$c.log; echo
done
timeout 600 python bench.py --router balanced --steps 10 --warmup 3 --skip-cpu > gpurun_out/bench_c2_balanced.log 2>&1
head -c 200 gpurun_out/bench_c2_balanced.log; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
head -c 300 gpurun_out/bench_reference.log; echo
