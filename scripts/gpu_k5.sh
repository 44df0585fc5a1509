cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/k5c.txt; : > $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export ES_JIT_CACHE=0
for b in 300 1000 3000; do echo "BAR=$b" >> $O; ES_K1_BAR=$b timeout 600 python scripts/probe_k1var.py 5 256 >> $O 2>&1; done
echo "BAR=1000 R=230" >> $O; ES_K1_BAR=1000 ES_K1_SPILL_R=230 timeout 600 python scripts/probe_k1var.py 5 256 >> $O 2>&1
for b in 300 1000; do echo "k4 BAR=$b" >> $O; ES_K1_BAR=$b timeout 600 python scripts/probe_k1var.py 4 256 >> $O 2>&1; done
