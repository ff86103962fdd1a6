set -u
TAG=r02_v5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in c2 c3 c4; do
  CMD="env DPR_STEP_LOOP=host python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_launches_${c}.csv $CMD > /dev/null 2>&1; echo "launches $c rc=$?"
done
bash tools/ncu_capture.sh $TAG c2 regex:k_trace 2 2 "k_trace_path k_trace_occl"
bash tools/ncu_capture.sh $TAG c3 "regex:k_trace_path|k_march_occl" 2 2 "k_trace_path k_march_occl"
bash tools/ncu_capture.sh $TAG c4 regex:k_trace_path 0 8 "k_trace_path"
