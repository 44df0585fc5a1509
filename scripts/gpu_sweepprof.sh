cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_sass_gpu.py tests/test_sweep_gpu.py -x -q > gpurun_out/sass_gpu2.log 2>&1
ES_VERBOSE=1 timeout 600 python scripts/profile_sweep_cold.py > gpurun_out/sweep_prof.txt 2> gpurun_out/sweep_prof.err
export ES_JIT_CACHE=0
timeout 300 python scripts/probe_direct.py one mult16 none -1 > gpurun_out/direct4.txt 2>&1
timeout 300 python scripts/probe_direct.py auto fault >> gpurun_out/direct4.txt 2>&1
