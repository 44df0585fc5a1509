"""Multi-rank host logic of the sharded sweep, on CPU with gloo (world 2).

Each rank runs the real schedule (shard.sharded_loop / rank_chunks, the same
rule es_session_launch applies on the GPU) with the kernel replaced by its
bit-exact CPU model (es_map_eval) and the skip rule of k1_skeleton.cu
(a chunk starting above the current minimum is not claimed); the MIN
all-reduce goes over gloo.  The combined answer must be the reference's
minimum-index witness.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_06627_b200 import shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, chunk_log2, slices, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_06627_b200 import es
    from tests.golden import recipes

    out = []
    for kind, spec in cases:
        x = recipes.build_random(spec) if kind == "random" else recipes.build_miter_recipe(spec)
        p = es.compile_program(x)
        n = x.num_pis
        total_words = 1 << max(n - 5, 0)
        cw = min(1 << chunk_log2, total_words)
        n_chunks = total_words // cw
        best = torch.tensor([1 << n], dtype=torch.int64)
        swept = []

        def launch(lo, hi):
            for c in shard.rank_chunks(lo, hi, rank, world):
                if (c * cw) << 5 > int(best.item()):
                    continue  # skip rule of the kernel's chunk claim
                swept.append(c)
                words = es.map_eval(p, c * cw, cw)
                nz = words.nonzero()[0]
                if len(nz):
                    w = int(nz[0])
                    v = int(words[w])
                    idx = ((c * cw + w) << 5) | ((v & -v).bit_length() - 1)
                    best[0] = min(int(best[0]), idx)

        def reduce():
            dist.all_reduce(best, op=dist.ReduceOp.MIN)

        shard.sharded_loop(n_chunks, slices, launch, reduce)
        allswept = [None] * world
        dist.all_gather_object(allswept, swept)
        out.append((int(best.item()), sorted(c for s in allswept for c in s), n_chunks))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_rank_chunks_partition():
    for world in (1, 2, 3, 8):
        for lo, hi in ((0, 17), (5, 40), (7, 8)):
            got = sorted(c for r in range(world) for c in shard.rank_chunks(lo, hi, r, world))
            assert got == list(range(lo, hi))
    assert shard.slice_bounds(10, 4) == [0, 2, 5, 7, 10]
    assert shard.slice_bounds(3, 8) == [0, 1, 2, 3]


@pytest.mark.parametrize("slices", [1, 4])
def test_gloo_two_ranks_min_index(golden, slices):
    from tests.golden import recipes

    specs = {s["name"]: s for s in recipes.miter_population()}
    rows = [("random", g) for g in golden["random"] if 12 <= g["num_pis"] <= 16][:12]
    rows += [("miter", specs[g["name"]]) for g in golden["miters"]
             if g["num_pis"] <= 16 and g["name"].startswith(("mult8_array_diagonal_mut",
                                                             "adder8", "mult8_array_booth"))]
    expect = {}
    for g in golden["random"]:
        expect[("random", g["seed"], g["pop"])] = g
    gm = {g["name"]: g for g in golden["miters"]}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, 4, slices, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for (kind, spec), (best, swept, n_chunks) in zip(rows, out):
        g = expect[("random", spec["seed"], spec["pop"])] if kind == "random" else gm[spec["name"]]
        n = g["num_pis"]
        want = g["witness_index"]
        got = None if best >= 1 << n else best
        assert got == want, (kind, spec)
        assert len(swept) == len(set(swept))  # no chunk swept twice
        if want is None:
            assert swept == list(range(n_chunks))  # EQ: full coverage
        else:  # every chunk below the witness's chunk was swept
            cw_patterns = (1 << n) // n_chunks
            assert set(range(want // cw_patterns + 1)) <= set(swept)
