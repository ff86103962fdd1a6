set -u
TAG=r02_v4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_${c}.json 2> gpurun_out/${TAG}_bench_${c}.err; echo "bench $c rc=$?"
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_launches_${c}.csv $CMD > /dev/null 2>&1; echo "launches $c rc=$?"
done
bash tools/ncu_capture.sh $TAG c2 regex:k_trace 2 2 "k_trace_path k_trace_occl"
bash tools/ncu_capture.sh $TAG c3 "regex:k_trace_path|k_march_occl" 2 2 "k_trace_path k_march_occl"
bash tools/ncu_capture.sh $TAG c4 regex:k_trace_path 0 8 "k_trace_path"
bash tools/ncu_capture.sh $TAG c4b "regex:k_collapse_r|k_agglo_p|k_permute_prims|k_scatter_c|k_part_prims|k_gather_prims" 0 24 "k_collapse_r k_agglo_p k_permute_prims" python tools/build_only.py c4 1
