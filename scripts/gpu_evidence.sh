#!/bin/bash
# Round evidence on one GPU: tests, full bench (with CPU baseline), per-op DRAM
# traffic of one forward, launch list, and ncu --set full captures of the hot
# kernels. Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -m paper_2306_06446_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/traffic.csv \
  python scripts/profile_forward.py --record gpurun_out/op_calls.json > gpurun_out/traffic.log 2>&1
# north-star kernels standalone at the bench shape (K1, K2a, K3, K5)
for k in sign_hash_stream_kernel binattn_fused tc_gemm_kernel mlp_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    --profile-from-start off -o gpurun_out/full_$k -f python scripts/kernels_standalone.py \
    > gpurun_out/ncu_full_$k.log 2>&1
done
# the forward's fused kernels (first launch inside the profiled forward)
for k in qkv_kernel ln_route_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 \
    --profile-from-start off -o gpurun_out/full_$k -f python scripts/profile_forward.py --warm 1 \
    > gpurun_out/ncu_full_$k.log 2>&1
done
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
head -c 400 gpurun_out/bench.log; echo
