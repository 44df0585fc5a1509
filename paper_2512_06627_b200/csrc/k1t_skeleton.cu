// k1t_skeleton.cu -- K1T: K1 with the word-uniform sub-network transposed
// across iterations (sm_100a).  Compiled to PTX at build time; the host
// splices two generated bodies (es_codegen_t.cpp) at ES_BODY_T1 / ES_BODY_T2.
//
// A node whose support avoids PIs 1..5 has the same value in all 32 bits of a
// word ("word-uniform"): K1 recomputes it in every lane of every iteration.
// Here each warp handles blocks of ES_TB iterations (32 words each):
//   phase 1: lane q (mod ES_TB) evaluates the word-uniform nodes for iteration
//            q of the block as a super-word (bit L = value for word 32*wb_q+L:
//            PIs 6..10 are lane-pattern constants, PIs 11.. bits of wb_q) and
//            stores the ones the per-lane logic consumes to shared memory;
//   phase 2: for each iteration q, every lane reads those super-words
//            (broadcast loads) and extracts its own bit as a full-word mask
//            with two FMA-pipe multiplies, then runs the per-lane LUTs.
// The uniform sub-network costs 1/ES_TB of its K1 issue count.
//
// Chunk claiming, minimum-index early exit and the warp ballot + atomicMin
// are K1's (k1_skeleton.cu).

#ifndef ES_TB
#define ES_TB 16
#endif

struct K1Params {
    unsigned long long *best;
    unsigned int *counter;
    unsigned long long first_chunk;
    unsigned long long n_slots;
    unsigned long long world;
    unsigned long long total_words;
    unsigned int chunk_log2;       // >= log2(32 * ES_TB * warps per CTA)
    unsigned int valid_mask;
    unsigned int one;              // == 1; opaque to ptxas (keeps the FMA-pipe extraction)
    unsigned int region_bytes;     // K1T: shared bytes per warp (boundary super-words)
    unsigned int cof_n;            // unused here (no cofactor copies)
    unsigned int cof_pos[8];
};

extern "C" __global__ void __launch_bounds__(ES_THREADS)
es_k1t(const K1Params p)
{
    extern __shared__ unsigned s_uni[];  // per warp: n_boundary x ES_TB super-words
    __shared__ unsigned long long s_chunk;
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const unsigned nwarps = ES_THREADS / 32;
    const unsigned pow2 = 1u << (31u - lane);
    const unsigned q1 = lane % ES_TB;
    // shared byte addresses: this warp's region; lane q1's column
    const unsigned region = (unsigned)__cvta_generic_to_shared(s_uni) + warp * p.region_bytes;
    const unsigned s_store = region + q1 * 4u;
    for (;;) {
        if (threadIdx.x == 0) {
            unsigned long long c = ~0ull;
            const unsigned long long k = atomicAdd(p.counter, 1u);
            if (k < p.n_slots) {
                c = p.first_chunk + k * p.world;
                const unsigned long long first_pattern = (c << p.chunk_log2) << 5;
                if (first_pattern > *(volatile unsigned long long *)p.best) c = ~0ull;
            }
            s_chunk = c;
        }
        __syncthreads();
        const unsigned long long chunk = s_chunk;
        __syncthreads();
        if (chunk == ~0ull) break;
        const unsigned long long w0 = chunk << p.chunk_log2;
        const unsigned words = 1u << p.chunk_log2;
#pragma unroll 1
        for (unsigned blk = warp * 32u * ES_TB; blk < words; blk += nwarps * 32u * ES_TB) {
            const unsigned long long wb0 = (w0 + blk) >> 5;  // first word-block of this block
            {   // phase 1: word-uniform super-words for iteration q1
                const unsigned long long wbq = wb0 + q1;
                asm volatile("// ES_BODY_T1 %0 %1 %2"
                             :: "r"((unsigned)wbq), "r"((unsigned)(wbq >> 32)), "r"(s_store)
                             : "memory");
            }
            __syncwarp();
#pragma unroll 1
            for (unsigned q = 0; q < ES_TB; ++q) {  // phase 2
                const unsigned long long wb = wb0 + q;
                const unsigned long long w = (wb << 5) | lane;
                unsigned out;
                asm volatile("// ES_BODY_T2 %0 %1 %2 %3 %4 %5 %6"
                             : "=r"(out)
                             : "r"((unsigned)wb), "r"((unsigned)(wb >> 32)), "r"(lane), "r"(pow2),
                               "r"(p.one), "r"(region + q * 4u)
                             : "memory");
                out &= p.valid_mask;
                if (w >= p.total_words) out = 0u;
                const unsigned hit = __ballot_sync(0xffffffffu, out != 0u);
                if (hit) {
                    const int l = __ffs(hit) - 1;
                    const unsigned o = __shfl_sync(0xffffffffu, out, l);
                    if (lane == 0)
                        atomicMin_system(p.best, (((wb << 5) | (unsigned)l) << 5) | (unsigned long long)(__ffs(o) - 1));
                }
            }
            __syncwarp();
        }
    }
}
