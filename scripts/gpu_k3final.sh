cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/k3final.txt; : > $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider >> $O 2>&1; echo "pytest gpu exit $?" >> $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $O 2>&1; echo "smoke exit $?" >> $O
for i in 1 2; do timeout 300 python scripts/probe_sim.py 64 4096 16384 65536 >> $O 2>&1; done
