#!/bin/bash
# Full evidence refresh for one tag (under gpurun, from the repo root):
#   bash tools/refresh_round.sh TAG
# Bench lines of every workload + the reference arm (tools/bench_all.sh), then per configs[1],
# configs[2], configs[3]: the ncu launch list of one host-loop step and an ncu --set full
# capture of the trace / march kernels exported to CSV (tools/ncu_capture.sh), and configs[3]'s
# LBVH build kernels under ncu.  Every ncu command runs after the same command exited 0 alone.
TAG=$1
mkdir -p gpurun_out
bash tools/bench_all.sh $TAG
export DPR_STEP_LOOP=host
for C in c2 c3 c4; do
  CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/plain_l_$C.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches_$C.csv $CMD > gpurun_out/ncu_launches_$C.log 2>&1
  echo "launches $C rc=$?"
done
bash tools/ncu_capture.sh $TAG c2 "regex:k_trace" 2 2 "k_trace_occl k_trace_path"
bash tools/ncu_capture.sh $TAG c3 "regex:k_trace|k_march" 2 3 "k_trace_path k_march_occl"
bash tools/ncu_capture.sh $TAG c4 "regex:k_trace_path" 0 8 "k_trace_path"
bash tools/ncu_capture.sh $TAG c4b "regex:k_collapse_r|k_agglo_p|k_permute_prims|k_scatter_w|k_part_prims|k_gather_prims|k_tile_hist|k_morton_h" 0 30 "k_collapse_r k_agglo_p" python tools/build_only.py c4 1
# ncu source pages run to tens of MB: compressed so gpurun_out stays under the return cap
find gpurun_out -name "${TAG}_*.csv" -size +1M -exec gzip -f {} \;
ls -la gpurun_out | grep $TAG
