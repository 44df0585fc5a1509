cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export ES_JIT_CACHE=0
for c in ${COSTS:-1.0 0.8 0.7 0.5}; do ES_IMAD_COST=$c timeout 300 python scripts/probe_imad.py ${KS:-4}; done > gpurun_out/probe_imad.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cofactor_gpu.py tests/test_split_gpu.py -q -x -m gpu > gpurun_out/probe_imad_tests.txt 2>&1
