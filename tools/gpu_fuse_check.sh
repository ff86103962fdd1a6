set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_fuse.log 2>&1
tail -3 gpurun_out/pytest_fuse.log
for i in 1 2; do
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/fuse_on_c2_$i.json 2>gpurun_out/fuse_on_c2.err
DPR_NO_FUSE_RESOLVE=1 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/fuse_off_c2_$i.json 2>/dev/null
done
timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/fuse_on_c3.json 2>/dev/null
DPR_NO_FUSE_RESOLVE=1 timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/fuse_off_c3.json 2>/dev/null
