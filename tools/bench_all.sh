#!/bin/bash
# Bench lines of every workload for one tag (under gpurun, from the repo root):
#   bash tools/bench_all.sh TAG   -> gpurun_out/TAG_bench_{c1,c2,c3,c3_delta,c4,c5,reference_arm}.json
TAG=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for C in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_${C}.json 2> gpurun_out/${TAG}_bench_${C}.err
  echo "$C rc=$?"
done
timeout 600 python bench.py --config c3 --flags 16 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c3_delta.json 2>/dev/null; echo "c3 delta rc=$?"
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2>/dev/null; echo "c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference_arm.json 2>/dev/null; echo "ref rc=$?"
