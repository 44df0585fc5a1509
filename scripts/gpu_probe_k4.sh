cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ES_VERBOSE=1 timeout 300 python scripts/probe_k4.py > gpurun_out/probe_k4_verbose.txt 2>&1
for o in ${ITEMS:-4096}; do echo "item $o"; ES_K4_ITEM=$o timeout 300 python scripts/probe_k4.py; ES_K4_ITEM=$o timeout 300 python scripts/probe_k4_sweep.py 2>&1 | head -1; done > gpurun_out/probe_k4.txt 2>&1
timeout 900 python -m pytest tests/test_config4_gpu.py tests/test_k4_gpu.py -q -x > gpurun_out/probe_k4_tests.txt 2>&1
