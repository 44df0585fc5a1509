cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:es_k4 -s 30 -c 1 -o /tmp/k4_full2 -f python scripts/ncu_cones_k4.py > gpurun_out/ncu_k4_full2.log 2>&1
ls -la /tmp/k4_full2.ncu-rep >> gpurun_out/ncu_k4_full2.log
ncu -i /tmp/k4_full2.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/k4_source.csv.gz
python scripts/ncu_summary.py /tmp/k4_full2.ncu-rep gpurun_out/k4_full2_summary.json > /dev/null 2>&1
ls -la gpurun_out >> gpurun_out/ncu_k4_full2.log
