"""Search single-gate faults (AND<->XOR flips) of the config miters whose
minimum-index counterexample is deep, using the CPU oracle on all cores.
The chosen gate indices go into recipes.DEEP_FAULTS; make_golden.py then pins
their witnesses by running the reference itself (workers=1)."""
import random
import sys
import time

from oracle import oracle as O
from paper_2512_06627_b200 import miter as M


def main(width: int, arch: str, want_log2: int, tries: int, seed: int = 1) -> None:
    m = M.gen_multiplier_miter(width, "array", arch)
    rng = random.Random(seed)
    n = m.num_pis
    lo_batches = 1 << max(0, want_log2 - 14)
    found = []
    for _ in range(tries):
        gi = rng.randrange(len(m.gates))
        p = O.compile_program(M.flip_gate(m, gi))
        t = time.time()
        v, idx, _ = O.min_witness(p, max_batches=lo_batches)
        if v == O.ES_COUNTEREXAMPLE:
            continue  # shallow
        v, idx, _ = O.min_witness(p)
        print(f"gate {gi}: {v} idx={idx} ({idx.bit_length() if idx else '-'} bits) "
              f"{time.time() - t:.1f}s", flush=True)
        if v == O.ES_COUNTEREXAMPLE:
            found.append((gi, idx))
    print(width, arch, found)


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
