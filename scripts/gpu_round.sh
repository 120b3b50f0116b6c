#!/bin/bash
# GPU round-trip: build, tests, bench, launch list, and one `ncu --set full`
# capture per hot kernel (single GPU; never a multi-rank command).
set -u
mkdir -p gpurun_out
bash scripts/gpu_check.sh
for k in ${NCU_KERNELS:-mlp_kernel attn_out_band_kernel tc_gemm_kernel sign_hash_stream_kernel kv_partial_kernel route_kernel ln_route_kernel}; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    --profile-from-start off -o gpurun_out/full_$k -f python scripts/profile_forward.py --warm 1 \
    > gpurun_out/ncu_full_$k.log 2>&1
  echo "ncu $k: $?"
done
