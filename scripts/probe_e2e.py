import sys, time, os
sys.path.insert(0, '.')
import bench
import torch
torch.cuda.init()
r = bench.measure_other_configs(0)
print("before", {k: round(v["e2e_ms"], 2) for k, v in r.items()})
print(bench.disk_cache_ttv("mult16", "auto"))
r = bench.measure_other_configs(0)
print("after", {k: round(v["e2e_ms"], 2) for k, v in r.items()})
