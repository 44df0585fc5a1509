cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export ES_JIT_CACHE=0
timeout 900 ncu --set full --clock-control none -k regex:es_k1 -s 2 -c 1 -o gpurun_out/k1_k4 -f python scripts/ncu_k1k.py 4 > gpurun_out/ncu_k4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:es_k1 -s 2 -c 1 -o gpurun_out/k1_k5 -f python scripts/ncu_k1k.py 5 > gpurun_out/ncu_k5.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:es_k1 -s 2 -c 1 -o gpurun_out/k1_k4d -f python scripts/ncu_k1k.py 4 -1 > gpurun_out/ncu_k4d.log 2>&1
