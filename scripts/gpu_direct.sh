cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for k in 0 2; do timeout 60 python scripts/dbg_direct.py $k >> gpurun_out/dbg8.txt 2>&1; done
timeout 900 python -m pytest tests/test_sass_gpu.py -x -q > gpurun_out/sass_gpu.log 2>&1
timeout 900 python scripts/probe_direct.py > gpurun_out/probe_direct.txt 2>&1
