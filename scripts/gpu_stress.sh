cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/stress2.txt; : > $O
timeout 1500 python scripts/stress_parity.py 1200 21 12 27 600 >> $O 2>&1
timeout 1200 python scripts/stress_parity.py 300 22 26 36 1500 >> $O 2>&1
timeout 900 python scripts/stress_parity.py 300 23 6 14 200 >> $O 2>&1
