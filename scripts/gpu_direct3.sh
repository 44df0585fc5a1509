cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/direct3.txt; : > $O
export ES_JIT_CACHE=0
for w in 8 24 64; do for r in 96 200; do echo "W=$w R=$r" >> $O; ES_SASS_WINDOW=$w ES_SASS_REMAT=$r timeout 300 python scripts/probe_direct.py one mult16 4 -1 >> $O 2>&1; done; done
