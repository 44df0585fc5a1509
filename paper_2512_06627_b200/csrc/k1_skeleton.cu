// k1_skeleton.cu -- K1, the straight-line exact-simulation kernel (sm_100a).
//
// Compiled at BUILD time to PTX (nvcc -ptx -arch=compute_100a); at run time
// the host splices the per-program LOP3 body (es_compile.cpp:emit_body_ptx)
// in place of the ES_BODY marker and compiles the result to SASS with the
// in-process PTX compiler (es_jit.cpp).  Everything around the body is
// hand-written here:
//
//  * persistent CTAs claim chunks of 2^chunk_log2 words in increasing order
//    from a device counter (load balance + monotone order for early exit);
//  * one thread evaluates one 32-pattern word per iteration, lanes of a warp
//    take consecutive words, so the lowest set ballot lane is the warp's
//    minimum failing word;
//  * a failing word is folded into the global minimum with one 64-bit
//    atomicMin per warp (replaces es.py:317-321's lock + stop cell);
//  * a CTA stops claiming once the next chunk starts above the current
//    minimum, so every chunk below the final minimum is fully evaluated and
//    the answer equals the reference's workers=1 witness (es.py:297-320).
//
// Multi-GPU: chunk ids of one launch are first_chunk + k*world, k < n_slots
// (the host puts this rank's residue class in first_chunk).  `best` is the
// rank-local copy of the global minimum, reduced across ranks between
// launches.

struct K1Params {
    unsigned long long *best;      // min failing pattern, sentinel 2^n
    unsigned int *counter;         // chunk claim counter, zeroed before launch
    unsigned long long first_chunk;
    unsigned long long n_slots;    // chunks this launch may claim
    unsigned long long world;      // chunk stride between claims
    unsigned long long total_words;
    unsigned int chunk_log2;       // words per chunk = 2^chunk_log2 (>= blockDim)
    unsigned int valid_mask;       // pattern bits of a word that exist (n < 5)
    unsigned int one;              // == 1, opaque to ptxas (IMAD coefficients)
    unsigned int region_bytes;     // K1T: shared bytes per warp (boundary super-words)
};

extern "C" __global__ void __launch_bounds__(ES_THREADS)
es_k1(const K1Params p)
{
    __shared__ unsigned long long s_chunk;
    const unsigned lane = threadIdx.x & 31u;
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
        for (unsigned it = 0; it < words; it += ES_THREADS) {
            const unsigned long long w = w0 + it + threadIdx.x;
            unsigned out;
            asm volatile("// ES_BODY %0 %1 %2 %3"
                         : "=r"(out) : "r"((unsigned)w), "r"((unsigned)(w >> 32)), "r"(p.one));
            out &= p.valid_mask;
            if (w >= p.total_words) out = 0u;
            const unsigned hit = __ballot_sync(0xffffffffu, out != 0u);
            if (hit) {
                const int l = __ffs(hit) - 1;
                const unsigned o = __shfl_sync(0xffffffffu, out, l);
                const unsigned long long wl = __shfl_sync(0xffffffffu, w, l);
                // system scope: `best` may be a peer GPU's word mapped over NVLink (CUDA IPC)
                if (lane == 0) atomicMin_system(p.best, (wl << 5) | (unsigned long long)(__ffs(o) - 1));
            }
        }
    }
}
