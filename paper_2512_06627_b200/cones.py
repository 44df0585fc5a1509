"""Sub-miter extraction: the sweep's candidate node pairs as ES jobs.

Harness for BASELINE.json config 4 ("~10k internal node-pair cones of 14-24
PIs drawn from a 16x16 multiplier miter, batched ES jobs") and the first
piece of SURVEY 8(f) next-1/next-2 (the sweep's sub-miter stream).

* ``simulate``       -- word-parallel random simulation (sim.py:15-38)
* ``candidate_classes`` -- canonical signatures and PE classes
                        (sweep.py:54-81: complements share a key)
* ``extract_submiter``  -- cone-local miter of a == b ^ polarity with dense
                        PI renumbering and merge-map collapsing
                        (sweep.py:92-158)
* ``config4_cones``  -- deterministic ~10k-cone workload.
"""

from __future__ import annotations

import ctypes
import random
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .xag import FALSE, Gate, GateKind, Lit, Xag, XagBuilder, packed_gates

_ONES = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclass
class SubMiter:
    """Localized equivalence obligation (sweep.py:44-51)."""

    circuit: Xag
    origin: tuple[int, int]
    merged_history: dict = field(default_factory=dict)
    pi_map: tuple[int, ...] = ()
    id: int = 0


def simulate(xag, words: int, seed: int) -> np.ndarray:
    """Node value words under seeded random PI words (sim.py:15-38)."""
    rng = np.random.default_rng(seed)
    vals = np.zeros((1 + xag.num_pis + len(xag.gates), words), dtype=np.uint64)
    vals[1:xag.num_pis + 1] = rng.integers(0, 1 << 64, size=(xag.num_pis, words),
                                           dtype=np.uint64)
    base = 1 + xag.num_pis
    for i, g in enumerate(xag.gates):
        a = vals[g.in0.node] ^ _ONES if g.in0.neg else vals[g.in0.node]
        b = vals[g.in1.node] ^ _ONES if g.in1.neg else vals[g.in1.node]
        vals[base + i] = (a & b) if g.kind == GateKind.AND else (a ^ b)
    return vals


def candidate_classes(xag, words: int = 1, seed: int = 0) -> list[list[tuple[int, bool]]]:
    """PE classes from canonical signatures min(raw, ~raw) (sweep.py:54-81)."""
    vals = simulate(xag, words, seed)
    groups: dict[bytes, list[tuple[int, bool]]] = {}
    for node in range(1 + xag.num_pis, vals.shape[0]):
        raw = vals[node].tobytes()
        inv = (vals[node] ^ _ONES).tobytes()
        key, pol = (inv, True) if inv < raw else (raw, False)
        groups.setdefault(key, []).append((node, pol))
    return [sorted(g) for g in groups.values() if len(g) >= 2]


def _resolve(node: int, merges: dict[int, Lit]) -> tuple[int, bool]:
    neg = False
    while node in merges:
        rep = merges[node]
        node, neg = rep.node, neg != rep.neg
    return node, neg


def support(xag, node: int, merges: dict[int, Lit] | None = None) -> set[int]:
    merges = merges or {}
    out, seen, stack = set(), set(), [node]
    while stack:
        v = stack.pop()
        if v in seen or v == 0:
            continue
        seen.add(v)
        if v <= xag.num_pis:
            out.add(v)
            continue
        g = xag.gates[v - 1 - xag.num_pis]
        stack.append(_resolve(g.in0.node, merges)[0])
        stack.append(_resolve(g.in1.node, merges)[0])
    return out


def support_masks(xag) -> list[int]:
    """Structural support of every node as a PI bitmask (bit j-1 = PI j)."""
    sup = [0] * (1 + xag.num_pis + len(xag.gates))
    for j in range(1, xag.num_pis + 1):
        sup[j] = 1 << (j - 1)
    base = 1 + xag.num_pis
    for i, g in enumerate(xag.gates):
        sup[base + i] = sup[g.in0.node] | sup[g.in1.node]
    return sup


def extract_submiter(xag, a: int, b: int, merges: dict[int, Lit] | None = None,
                     polarity: bool = False, sm_id: int = 0) -> SubMiter:
    """Cone-local miter for a == b ^ polarity (sweep.py:92-158)."""
    merges = merges or {}
    an, aneg = _resolve(a, merges)
    bn, bneg = _resolve(b, merges)
    sup = support(xag, an, merges) | support(xag, bn, merges)
    pi_map = tuple(sorted(sup))
    pi_index = {orig: i + 1 for i, orig in enumerate(pi_map)}
    bld = XagBuilder(len(pi_map))
    memo: dict[int, Lit] = {0: FALSE}

    def mapped(lit: Lit) -> Lit:
        node, neg = _resolve(lit.node, merges)
        got = memo[node]
        return Lit(got.node, got.neg ^ neg ^ lit.neg)

    seen: set[int] = set()
    stack = [(an, False), (bn, False)]
    while stack:
        node, expanded = stack.pop()
        if node == 0 or node in memo:
            continue
        if node <= xag.num_pis:
            memo[node] = bld.pi(pi_index[node])
            continue
        g = xag.gates[node - 1 - xag.num_pis]
        if expanded:
            l0, l1 = mapped(g.in0), mapped(g.in1)
            memo[node] = bld.add_and(l0, l1) if g.kind == GateKind.AND else bld.add_xor(l0, l1)
            continue
        if node in seen:
            continue
        seen.add(node)
        stack.append((node, True))
        stack.append((_resolve(g.in0.node, merges)[0], False))
        stack.append((_resolve(g.in1.node, merges)[0], False))
    la = Lit(memo[an].node, memo[an].neg != aneg)
    lb = Lit(memo[bn].node, memo[bn].neg != bneg)
    out = bld.add_xor(la, lb)
    if polarity:
        out = ~out
    return SubMiter(bld.finish([out]), (a, b), dict(merges), pi_map, sm_id)


class NativeBatch:
    """Sub-miters extracted and compiled in C++ (es_batch_extract), ready for
    one batched device sweep.  Extraction is extract_submiter's
    (sweep.py:92-158) step for step; programs are the reference schedule."""

    def __init__(self, parent, pairs, merges: dict[int, Lit] | None = None, threads: int = 0):
        pairs = list(pairs)
        n, g = parent.num_pis, len(parent.gates)
        kind, in0, in1 = packed_gates(parent)
        merges = merges or {}
        mn = np.array(list(merges.keys()), np.int32)
        ml = np.array([l.node * 2 + int(l.neg) for l in merges.values()], np.uint32)
        a = np.array([p[0] for p in pairs], np.int32)
        b = np.array([p[1] for p in pairs], np.int32)
        pol = np.array([int(p[2]) if len(p) > 2 else 0 for p in pairs], np.uint8)
        h = ctypes.c_void_p()
        N.check(N.lib().es_batch_extract(n, g, kind.ctypes.data, in0.ctypes.data, in1.ctypes.data,
                                         len(mn), mn.ctypes.data, ml.ctypes.data, len(pairs),
                                         a.ctypes.data, b.ctypes.data, pol.ctypes.data, threads,
                                         ctypes.byref(h)))
        self._h = h
        self.parent_pis = n
        self.origins = [(int(p[0]), int(p[1])) for p in pairs]

    def __len__(self) -> int:
        return N.lib().es_batch_size(self._h)

    def info(self, i: int) -> dict:
        v = [ctypes.c_int32() for _ in range(5)]
        hsh = ctypes.c_uint64()
        rc = N.lib().es_batch_info(self._h, i, ctypes.byref(v[0]), ctypes.byref(v[1]),
                                   ctypes.byref(hsh), ctypes.byref(v[2]), ctypes.byref(v[3]),
                                   ctypes.byref(v[4]))
        if rc not in (0, N.ES_E_TOO_MANY_INPUTS):
            N.check(rc)
        return {"num_pis": v[0].value, "num_gates": v[1].value, "hash": hsh.value,
                "num_instrs": v[2].value, "num_registers": v[3].value, "G": v[4].value,
                "eligible": rc == 0}

    def table(self) -> dict:
        """Per-job arrays: num_pis, num_gates, G, hash."""
        n = len(self)
        out = {"num_pis": np.zeros(n, np.int32), "num_gates": np.zeros(n, np.int32),
               "G": np.zeros(n, np.int32), "hash": np.zeros(n, np.uint64)}
        N.check(N.lib().es_batch_table(self._h, out["num_pis"].ctypes.data,
                                       out["num_gates"].ctypes.data, out["G"].ctypes.data,
                                       out["hash"].ctypes.data))
        return out

    def k2_stats(self) -> dict:
        """Per-job interpreter program shape (after prepare): num_slots,
        num_records, cofactor_pis; -1 where no program was built yet."""
        n = len(self)
        out = {k: np.zeros(n, np.int32) for k in ("num_slots", "num_records", "cofactor_pis")}
        N.check(N.lib().es_batch_k2_stats(self._h, out["num_slots"].ctypes.data,
                                          out["num_records"].ctypes.data,
                                          out["cofactor_pis"].ctypes.data))
        return out

    def k2_traffic(self) -> dict:
        """Per-job shared-memory slot loads and stores of one interpreter pass."""
        n = len(self)
        out = {k: np.zeros(n, np.int32) for k in ("loads", "stores")}
        N.check(N.lib().es_batch_k2_traffic(self._h, out["loads"].ctypes.data, out["stores"].ctypes.data))
        return out

    def submiter(self, i: int) -> SubMiter:
        inf = self.info(i)
        ng, n = inf["num_gates"], inf["num_pis"]
        kind = np.zeros(ng, np.uint8)
        in0 = np.zeros(ng, np.uint32)
        in1 = np.zeros(ng, np.uint32)
        pm = np.zeros(n, np.int32)
        out = ctypes.c_uint32()
        N.check(N.lib().es_batch_xag(self._h, i, kind.ctypes.data, in0.ctypes.data,
                                     in1.ctypes.data, ctypes.byref(out), pm.ctypes.data))
        gates = tuple(Gate(GateKind(int(k)), Lit.unpack(int(x)), Lit.unpack(int(y)))
                      for k, x, y in zip(kind, in0, in1))
        return SubMiter(Xag(n, gates, (Lit.unpack(out.value),)), self.origins[i] if
                        i < len(self.origins) else (0, 0), {}, tuple(int(q) for q in pm), i)

    def packed(self, i: int):
        """Sub-miter i as packed arrays: (num_pis, kind, in0, in1, out_lit)."""
        inf = self.info(i)
        ng, n = inf["num_gates"], inf["num_pis"]
        kind = np.zeros(ng, np.uint8)
        in0 = np.zeros(ng, np.uint32)
        in1 = np.zeros(ng, np.uint32)
        out = ctypes.c_uint32()
        N.check(N.lib().es_batch_xag(self._h, i, kind.ctypes.data, in0.ctypes.data,
                                     in1.ctypes.data, ctypes.byref(out), None))
        return n, kind, in0, in1, out.value

    def prepare(self, threads: int = 0) -> None:
        """Build every job's interpreter program now (cofactor depth, schedule);
        run_arrays would do it on its first call."""
        N.check(N.lib().es_batch_prepare(self._h, threads))

    def select(self, idx) -> None:
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        N.check(N.lib().es_batch_select(self._h, len(idx), idx.ctypes.data))
        self.origins = [self.origins[i] for i in idx]

    def run_arrays(self, budget: float | None = None, cancel=None, device: int = 0,
                   engine: str = "auto", cofactor="auto") -> np.ndarray:
        """Batched run_exhaustive over every sub-miter (witnesses re-checked on
        the sub-miter by the library); the raw es_result records as a numpy
        structured array (fields of include/es_b200.h es_result).  engine
        "auto": jobs of >= 2e12 gate-patterns get their own K1 kernel (JIT on
        parallel host threads), the rest share one K2 launch; "interp": all K2.
        cofactor "none": interpreter programs without the cofactor-depth search
        (cheaper on the host for batches with little device work)."""
        from .es import _CancelWatcher, _opts

        n = len(self)
        outs = (N.EsResult * n)()
        # budget <= 0 is decided natively, after each job's constant-rail check
        with _CancelWatcher(cancel) as cw:
            opts = _opts(device, engine, budget, cw.address, 20.0, 0, cofactor=cofactor)
            N.check(N.lib().es_batch_run(self._h, ctypes.byref(opts), outs))
        return np.ctypeslib.as_array(outs)

    def run(self, budget: float | None = None, cancel=None, device: int = 0, engine: str = "auto",
            cofactor="auto"):
        """As run_arrays, as a list of EsResult (None for ineligible jobs)."""
        from .es import _to_esresult

        outs = self.run_arrays(budget, cancel, device, engine, cofactor)
        pis = self.table()["num_pis"]
        res = []
        for i in range(len(outs)):
            rec = N.EsResult.from_buffer_copy(outs[i].tobytes())
            res.append(None if rec.reason == -1 else _to_esresult(rec, int(pis[i])))
        return res

    def extend(self, other: "NativeBatch") -> None:
        """Move all of ``other``'s sub-miters to the end of this batch."""
        N.check(N.lib().es_batch_merge(self._h, other._h))
        self.origins.extend(other.origins)
        other.origins = []

    def close(self) -> None:
        if self._h:
            N.lib().es_batch_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def config4_pairs(lo: int = 14, hi: int = 24, seed: int = 0, sim_words: int = 1,
                  rounds: int = 64):
    """Yield (miter, pairs) rounds: candidate pairs from short random
    simulations of 16x16 multiplier miters (sweep.py:318-345)."""
    from . import miter as M

    archs = [("array", "booth"), ("array", "wallace"), ("array", "diagonal"),
             ("diagonal", "booth"), ("wallace", "booth"), ("diagonal", "wallace")]
    rng = random.Random(seed)
    built: dict = {}
    for round_ in range(rounds):
        a_arch, b_arch = archs[round_ % len(archs)]
        if (a_arch, b_arch) not in built:  # deterministic: build each parent once
            mm = M.gen_multiplier_miter(16, a_arch, b_arch)
            built[(a_arch, b_arch)] = (mm, support_masks(mm))
        m, sup = built[(a_arch, b_arch)]
        pairs = []
        for cls in candidate_classes(m, sim_words, seed + round_ // len(archs)):
            nodes = [n for n, _ in cls if sup[n].bit_count() <= hi]
            pol = dict(cls)
            for i in range(len(nodes)):
                for j in range(i + 1, len(nodes)):
                    a, b = nodes[i], nodes[j]
                    if lo <= (sup[a] | sup[b]).bit_count() <= hi:
                        pairs.append((a, b, pol[a] != pol[b]))
        rng.shuffle(pairs)
        yield m, pairs


def config4_batches(count: int = 10_000, lo: int = 14, hi: int = 24, seed: int = 0,
                    threads: int = 0) -> list[NativeBatch]:
    """BASELINE.json config 4: ~10k distinct candidate-pair sub-miters with
    lo..hi PIs drawn from 16x16 multiplier miters -- the array-vs-Booth miter
    of configs[2] first, pooled with the other architecture pairs because one
    64-pattern simulation of one miter proposes only ~500 distinct cones in
    range.  Extraction and compilation run in C++ (es_batch_extract); the
    result is one NativeBatch per parent miter."""
    out: list[NativeBatch] = []
    seen: set[int] = set()
    total = 0
    t_pairs = t_extract = 0.0
    extracted = 0
    gen = config4_pairs(lo, hi, seed)
    while total < count:
        t = time.perf_counter()
        try:
            m, pairs = next(gen)
        except StopIteration:
            break
        t_pairs += time.perf_counter() - t
        t = time.perf_counter()
        nb = NativeBatch(m, pairs, threads=threads)  # C++ extract_submiter + compile_program
        t_extract += time.perf_counter() - t
        extracted += len(pairs)
        tab = nb.table()
        keep = []
        for i in range(len(nb)):
            h = int(tab["hash"][i])
            if not lo <= tab["num_pis"][i] <= hi or h in seen:
                continue
            seen.add(h)
            keep.append(i)
            if total + len(keep) >= count:
                break
        nb.select(keep)
        total += len(keep)
        out.append(nb)
    LAST_TIMING.clear()
    LAST_TIMING.update(pair_sampling_s=t_pairs, extract_compile_s=t_extract, pairs_extracted=extracted,
                       jobs=total)
    return out


# host time of the last config4_batches call: pair sampling (random simulation
# and candidate classes, the sweep's job; numpy here), and C++ extraction +
# reference-schedule compilation of every candidate pair (kept or not)
LAST_TIMING: dict = {}


def config4_batch(count: int = 10_000, lo: int = 14, hi: int = 24, seed: int = 0,
                  threads: int = 0) -> NativeBatch:
    """config4_batches merged into one batch (one device launch)."""
    bs = config4_batches(count, lo, hi, seed, threads)
    head = bs[0]
    for b in bs[1:]:
        head.extend(b)
    head.prepare(threads)
    return head


def sweep_round_batch(miter=None, words: int = 64, lo: int = 14, hi: int = 24, seed: int = 0,
                      threads: int = 0) -> NativeBatch:
    """The EQ-heavy variant of config 4: the candidate pairs the
    sweep itself sends after its 64-word random simulation (sweep.py:313-345)
    of ONE miter (default the configs[2] array-vs-Booth 16x16), every pair of
    a class whose cone has lo..hi PIs, distinct cones only.  A 64-word
    simulation leaves few false candidates, so most of these are EQ and must
    be swept completely."""
    from . import miter as M

    m = miter if miter is not None else M.gen_multiplier_miter(16, "array", "booth")
    sup = support_masks(m)
    pairs = []
    for cls in candidate_classes(m, words, seed):
        nodes = [n for n, _ in cls if sup[n].bit_count() <= hi]
        pol = dict(cls)
        for i in range(len(nodes)):
            for j in range(i + 1, len(nodes)):
                a, b = nodes[i], nodes[j]
                if lo <= (sup[a] | sup[b]).bit_count() <= hi:
                    pairs.append((a, b, pol[a] != pol[b]))
    nb = NativeBatch(m, pairs, threads=threads)
    tab = nb.table()
    seen, keep = set(), []
    for i in range(len(nb)):
        h = int(tab["hash"][i])
        if lo <= tab["num_pis"][i] <= hi and h not in seen:
            seen.add(h)
            keep.append(i)
    nb.select(keep)
    nb.prepare(threads)
    return nb


def config4_cones(count: int = 10_000, lo: int = 14, hi: int = 24, seed: int = 0):
    """The config-4 workload as Python SubMiters (tests, small counts)."""
    subs = []
    for nb in config4_batches(count, lo, hi, seed):
        subs.extend(nb.submiter(i) for i in range(len(nb)))
    return subs
