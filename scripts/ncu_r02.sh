set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_mult16.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_bench_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:es_k1 -s 2 -c 1 -o gpurun_out/r02_k1 python scripts/ncu_k1.py > gpurun_out/ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:es_k2 -c 3 -o gpurun_out/r02_k2 python scripts/ncu_cones.py > gpurun_out/ncu_k2.log 2>&1
ls -la gpurun_out
