"""Multi-rank sweeps on the GPU: 2 processes share cuda:0 (gloo for the
host barriers -- NCCL needs one GPU per rank).  Both exchanges:
  * p2p  : one minimum word in rank 0's memory, CUDA-IPC-mapped into every
           rank, kernel atomicMin + early exit (shard.sweep_peer);
  * nccl : per-slice MIN all-reduce of the rank-local word (shard.sweep_sharded).
Verdict, witness and patterns_evaluated must equal the reference's."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

# PI counts go down and up (16, 28, 24, 32, 24): one PeerBest must serve
# programs of any width (its words are armed with all-ones, not 2^n)
NAMES = ["adder8_ripple_lookahead_mut1", "mult14_array_diagonal", "mult12_array_wallace_flip1108",
         "mult16_array_booth_flip1220", "mult12_array_wallace"]


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_06627_b200 import es, shard
    from tests.golden import recipes

    specs = {s["name"]: s for s in recipes.miter_population()}
    peer = shard.PeerBest(None, 0) if mode == "p2p" else None
    out = []
    for name in NAMES:
        p = es.compile_program(recipes.build_miter_recipe(specs[name]))
        for _ in range(3):  # three times: every rotating word is re-armed and reused
            if peer is not None:
                r = shard.sweep_peer(p, peer, None, 0)
            else:
                r = shard.sweep_sharded(p, None, 0, slices=3)
        out.append((name, r.verdict, r.witness_index, r.patterns_evaluated))
    dist.barrier()
    if peer is not None:
        peer.close()
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["p2p", "nccl"])
def test_two_ranks_one_gpu(golden, gpu, mode):
    gm = {g["name"]: g for g in golden["miters"]}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, v, w, pe in out:
        g = gm[name]
        assert (v, w, pe) == (g["verdict"], g["witness_index"], g["patterns_evaluated"]), name
