cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/k3.txt; : > $O
timeout 900 python -m pytest tests/test_sim_gpu.py -x -q >> $O 2>&1
timeout 300 python scripts/probe_sim.py >> $O 2>&1
ES_SIM_LEVEL=1 timeout 300 python scripts/probe_sim.py >> $O 2>&1
