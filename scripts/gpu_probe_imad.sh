cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export ES_JIT_CACHE=0
for c in 1.0 0.7 0.5 0.4 0.3 0.2 0.1; do ES_IMAD_COST=$c timeout 300 python scripts/probe_imad.py 4 5; done > gpurun_out/probe_imad.txt 2>&1
