#!/bin/bash
# Full evidence refresh for one tag (under gpurun, from the repo root):
#   bash tools/refresh_round.sh TAG
# configs[1] and configs[2]: bench line + launch list + ncu --set full (tools/profile_round.sh);
# configs[0], configs[2] delta tracking, configs[3]: bench lines; the reference arm line.
TAG=$1
bash tools/profile_round.sh $TAG c2 regex:k_trace
bash tools/profile_round.sh $TAG c3
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c1.json 2>/dev/null; echo "c1 rc=$?"
timeout 600 python bench.py --config c3 --flags 16 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c3_delta.json 2>/dev/null; echo "c3 delta rc=$?"
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2>/dev/null; echo "c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference_arm.json 2>/dev/null; echo "ref rc=$?"
