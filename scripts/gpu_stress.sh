cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/stress.txt; : > $O
timeout 1500 python scripts/stress_parity.py 400 7 12 27 500 >> $O 2>&1
timeout 1200 python scripts/stress_parity.py 150 8 26 34 1200 >> $O 2>&1
