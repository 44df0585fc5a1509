cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/k2ctas.txt; : > $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 3 4; do echo "CTAS=$c" >> $O; ES_K2_CTAS=$c timeout 300 python scripts/probe_cones.py >> $O 2>&1; done
