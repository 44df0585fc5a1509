cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export ES_JIT_CACHE=0
for c in ${COSTS:-1.0 0.5}; do
  ES_IMAD_COST=$c timeout 900 ncu --set full --clock-control none --import-source on -k regex:es_k1 -s 2 -c 1 -o gpurun_out/k1_imad_$c -f python scripts/ncu_k1k.py 4 > gpurun_out/ncu_imad_$c.log 2>&1
done
