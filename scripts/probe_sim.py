"""Dev probe: K3 random simulation throughput (device-resident drive/output)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2512_06627_b200 import miter as M, sim
for words in [int(a) for a in sys.argv[1:]] or (64, 4096, 1 << 16):
    m = M.gen_multiplier_miter(16, "array", "booth")
    nn = 1 + m.num_pis + len(m.gates)
    pw = sim.random_pi_words(m.num_pis, words, 1)
    d_pi = torch.from_numpy(pw.view(np.int64)).cuda()
    d_out = torch.empty((nn, words), dtype=torch.int64, device="cuda")
    ds = sim.DeviceSim(m)
    st = torch.cuda.current_stream()
    for _ in range(3):
        ds.run(d_pi.data_ptr(), words, d_out.data_ptr(), st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        ds.run(d_pi.data_ptr(), words, d_out.data_ptr(), st.cuda_stream)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byts = (nn + m.num_pis) * words * 8
    gw = len(m.gates) * words * 64
    t = time.time(); cl = sim.pe_classes(m, words, 1); tc = time.time() - t
    print(f"words={words} nodes={nn} {ms:.3f}ms {byts / ms / 1e6:.0f} GB/s "
          f"{gw / ms * 1e3:.3e} gate-patterns/s  pe_classes {tc * 1e3:.1f}ms ({len(cl)} classes)", flush=True)
