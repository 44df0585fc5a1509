cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(timeout 600 python scripts/probe_k4_sweep.py; ES_K4=0 timeout 600 python scripts/probe_k4_sweep.py) > gpurun_out/probe_k4_sweep.txt 2>&1
