cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/direct2.txt; : > $O
timeout 900 python -m pytest tests/test_sass_gpu.py -x -q >> $O 2>&1
export ES_JIT_CACHE=0
for k in none 4; do timeout 300 python scripts/probe_direct.py one mult16 $k -1 >> $O 2>&1; ES_SASS_NO_REUSE=1 timeout 300 python scripts/probe_direct.py one mult16 $k -1 >> $O 2>&1; done
