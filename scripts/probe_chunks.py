"""Dev probe: K1 mult16 time vs chunk granularity, whole space and one 1/8 shard."""
import os, sys
sys.path.insert(0, '.')
import torch
from paper_2512_06627_b200 import es, shard, miter as M
m = M.gen_multiplier_miter(16, "array", "booth")
p = es.compile_program(m)
ts = [es.run_exhaustive(p, engine="jit", cofactor="throughput").stats["device_ms"] for _ in range(6)]
sess = shard.session_for(p, 0, "throughput")
best = torch.empty(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
sh = []
for rep in range(6):
    best.fill_(1 << 32)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sess.launch(st, best.data_ptr(), 0, sess.n_chunks, 3, 8); e1.record(); torch.cuda.synchronize()
    sh.append(e0.elapsed_time(e1))
print(f"per_cta={os.environ.get('ES_CHUNKS_PER_CTA', '64')} chunks={sess.n_chunks} full={min(ts[1:]):.3f}ms "
      f"shard1/8={min(sh[1:]):.3f}ms (ideal {min(ts[1:]) / 8:.3f})", flush=True)
