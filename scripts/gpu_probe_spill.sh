cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export ES_JIT_CACHE=0
P=gpurun_out/probe_spill2.txt; : > $P
for R in 140 150; do ES_K1_SPILL_R=$R ES_MAXNREG=168 timeout 200 python scripts/probe_k1var.py 4 128 >> $P 2>&1; done
ES_K1_SPILL_R=100 ES_MAXNREG=128 timeout 200 python scripts/probe_k1var.py 3 128 >> $P 2>&1
timeout 300 python scripts/probe_k1var.py 0 128 bfly >> $P 2>&1
timeout 300 python scripts/probe_k1var.py 0 256 bfly >> $P 2>&1
for R in 160 200 230; do ES_K1_SPILL_R=$R timeout 300 python scripts/probe_k1var.py 0 128 bfly >> $P 2>&1; done
ES_K1_SPILL_R=150 ES_MAXNREG=168 timeout 300 python scripts/probe_k1var.py 0 128 bfly >> $P 2>&1
ES_K1_SPILL_R=230 timeout 300 python scripts/probe_k1var.py 0 256 bfly >> $P 2>&1
