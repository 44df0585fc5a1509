cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/k2store.txt; : > $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/probe_cones.py >> $O 2>&1
timeout 900 python -m pytest tests/test_config4_gpu.py tests/test_cones.py tests/test_k2prog.py tests/test_gpu_parity.py tests/test_stress_gpu.py -x -q -m gpu >> $O 2>&1
