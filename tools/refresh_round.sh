#!/bin/bash
# Full evidence refresh for one tag (under gpurun, from the repo root):
#   bash tools/refresh_round.sh TAG
# configs[1], configs[2], configs[3]: bench line + launch list + ncu --set full of the trace
# kernels (tools/profile_round.sh); configs[0], configs[2] delta tracking, configs[4]: bench
# lines; the reference arm line; configs[3]'s LBVH build kernels under ncu.
TAG=$1
mkdir -p gpurun_out
bash tools/profile_round.sh $TAG c2 regex:k_trace
bash tools/profile_round.sh $TAG c3
NCU_SKIP=0 NCU_COUNT=8 bash tools/profile_round.sh $TAG c4 regex:k_trace_path
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c1.json 2>/dev/null; echo "c1 rc=$?"
timeout 600 python bench.py --config c3 --flags 16 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c3_delta.json 2>/dev/null; echo "c3 delta rc=$?"
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2>/dev/null; echo "c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference_arm.json 2>/dev/null; echo "ref rc=$?"
python tools/build_only.py c4 2 > gpurun_out/plain_b.log 2>&1 && ncu --set full --clock-control none --import-source on \
  -k "regex:k_collapse_r|k_agglo|k_permute_prims|k_scatter_c|k_part_prims|k_gather_prims" -c 24 \
  -o gpurun_out/${TAG}_build_c4 python tools/build_only.py c4 1 > gpurun_out/ncu_build.log 2>&1; echo "build ncu rc=$?"
