"""Config-4 K2 shared-memory model per launch group (W = words per thread),
to compare with ncu's l1tex__data_pipe_lsu_wavefronts_mem_shared_op_{ld,st}
per es_k2<W> launch: per warp and pass over a job's records, one broadcast
record load, `loads` slot loads and `stores` slot stores (incl. PI words) of
W wavefronts each."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2512_06627_b200 import cones  # noqa: E402

b = cones.config4_batch(10000)
res = b.run_arrays()
res = b.run_arrays()
st, tr = b.k2_stats(), b.k2_traffic()
ran = (res["reason"] != -1) & (res["engine"] == 2) & (st["num_records"] > 0)
W = np.maximum(res["regs_per_thread"], 1).astype(np.float64)
iters = res["patterns_swept"].astype(np.float64) / 32.0 / np.exp2(st["cofactor_pis"].astype(np.float64))
warp_iters = iters / (32.0 * W)
out = {}
for w in (1, 2, 4):
    m = ran & (W == w)
    out[f"W{w}"] = {"jobs": int(m.sum()),
                    "record_loads": float((warp_iters * (st["num_records"] + 1))[m].sum()),
                    "slot_load_wavefronts": float((warp_iters * tr["loads"] * W)[m].sum()),
                    "slot_store_wavefronts": float((warp_iters * tr["stores"] * W)[m].sum()),
                    "device_ms": float(res["device_ms"].max())}
print(json.dumps(out, indent=1))
