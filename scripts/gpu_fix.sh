cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export ES_JIT_CACHE=0
timeout 900 python scripts/probe_fix.py 28 4 > gpurun_out/fix.txt 2>&1
timeout 300 python scripts/probe_k1var.py 4 256 >> gpurun_out/fix.txt 2>&1
