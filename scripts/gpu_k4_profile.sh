cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --config cones --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_cones.json 2> gpurun_out/bench_cones.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cones.csv python scripts/ncu_cones_k4.py > gpurun_out/ncu_cones_list.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:es_k4 -s 20 -c 1 -o gpurun_out/k4_full -f python scripts/ncu_cones_k4.py > gpurun_out/ncu_k4_full.log 2>&1
