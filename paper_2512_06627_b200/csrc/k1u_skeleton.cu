// k1u_skeleton.cu -- K1U, the straight-line kernel with a warp-uniform
// "super-word" section (sm_100a).  Compiled to PTX at build time; the host
// splices the body (es_compile.cpp:emit_body_ptx_u) at ES_BODY_U.
//
// One warp per CTA and a static chunk schedule (chunk = first + k*world,
// k = blockIdx.x + i*gridDim.x), so the warp's word-block index wb -- which
// carries PIs 11.. -- is derived from blockIdx and loop counters only and is
// provably warp-uniform.  Lane L evaluates word w = 32*wb + L (PIs 6..10 =
// bits of L).  Every node whose support avoids PIs 1..10 is evaluated ONCE
// per warp as a super-word (bit L = lane L's value) from uniform operands, so
// ptxas can run it on the uniform datapath; lanes extract their bit with two
// FMA-pipe multiplies where such a node feeds the per-lane logic.  Chunks are
// visited in increasing order per CTA, so stopping at the first chunk above
// the current minimum keeps the minimum-index guarantee of K1.

struct K1Params {
    unsigned long long *best;
    unsigned int *counter;         // unused (static schedule)
    unsigned long long first_chunk;
    unsigned long long n_slots;
    unsigned long long world;
    unsigned long long total_words;
    unsigned int chunk_log2;
    unsigned int valid_mask;
    unsigned int one;              // == 1; opaque to ptxas (keeps the FMA-pipe extraction)
    unsigned int region_bytes;     // K1T: shared bytes per warp (boundary super-words)
    unsigned int cof_n;            // unused here (no cofactor copies)
    unsigned int cof_pos[8];
};

extern "C" __global__ void __launch_bounds__(32)
es_k1u(const K1Params p)
{
    const unsigned lane = threadIdx.x;
    const unsigned pow2 = 1u << (31u - lane);  // lane bit -> sign position (FMA-pipe extraction)
    const unsigned words = 1u << p.chunk_log2;
#pragma unroll 1
    for (unsigned long long k = blockIdx.x; k < p.n_slots; k += gridDim.x) {
        const unsigned long long chunk = p.first_chunk + k * p.world;
        if (((chunk << p.chunk_log2) << 5) > *(volatile unsigned long long *)p.best) break;
        const unsigned long long w0 = chunk << p.chunk_log2;
#pragma unroll 1
        for (unsigned it = 0; it < words; it += 32) {
            const unsigned long long wb = (w0 + it) >> 5;
            const unsigned long long w = (wb << 5) | lane;
            unsigned out;
            asm volatile("// ES_BODY_U %0 %1 %2 %3 %4 %5"
                         : "=r"(out)
                         : "r"((unsigned)wb), "r"((unsigned)(wb >> 32)), "r"(lane), "r"(pow2), "r"(p.one));
            out &= p.valid_mask;
            if (w >= p.total_words) out = 0u;
            const unsigned hit = __ballot_sync(0xffffffffu, out != 0u);
            if (hit) {
                const int l = __ffs(hit) - 1;
                const unsigned o = __shfl_sync(0xffffffffu, out, l);
                if (lane == 0) atomicMin_system(p.best, (((wb << 5) | (unsigned)l) << 5) | (unsigned long long)(__ffs(o) - 1));
            }
        }
    }
}
