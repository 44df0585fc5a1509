"""ncu target: one K3 random simulation of the mult16 miter (words = argv[1], default 65,536)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2512_06627_b200 import miter as M, sim
m = M.gen_multiplier_miter(16, "array", "booth")
words = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
pw = sim.random_pi_words(m.num_pis, words, 1)
d_pi = torch.from_numpy(pw.view(np.int64)).cuda()
d_out = torch.empty((1 + m.num_pis + len(m.gates), words), dtype=torch.int64, device="cuda")
ds = sim.DeviceSim(m)
for _ in range(3):
    ds.run(d_pi.data_ptr(), words, d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
