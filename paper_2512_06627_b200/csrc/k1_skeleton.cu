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
// Cofactor copies (es_cofactor.cpp, ES_MULTI): one iteration evaluates the
// 2^k words of one assignment each of the k cofactor PIs; the body returns
// the first failing copy's output word and its number, and the thread's word
// index w enumerates the other PIs only.  Pattern indices are
// rebuilt by inserting the cofactor bits (at pattern bits cof_pos[], PI-1):
// a chunk's first pattern (copy 0, its first w) is monotone in the chunk id,
// so the claim order and the skip rule keep the minimum-index guarantee.
//
// Multi-GPU: chunk ids of one launch are first_chunk + k*world, k < n_slots
// (the host puts this device's residue class in first_chunk).  `best` is one
// word in device 0's HBM that every GPU's kernels atomicMin into as peer
// memory (system scope), or a device-local copy combined by the host between
// launch slices when peer access is unavailable.

struct K1Params {
    unsigned long long *best;      // min failing pattern, sentinel 2^n
    unsigned int *counter;         // [0] claims, [1] chunks swept, [2] first slot hit_stop skipped
    unsigned long long first_chunk;
    unsigned long long n_slots;    // chunks this launch may claim
    unsigned long long world;      // chunk stride between claims
    unsigned long long hit_stop;   // stop claiming once *best < hit_stop (0: never)
    unsigned long long total_words;
    unsigned int chunk_log2;       // words per chunk = 2^chunk_log2 (>= blockDim)
    unsigned int valid_mask;       // pattern bits of a word that exist (n < 5)
    unsigned int one;              // == 1, opaque to ptxas (IMAD coefficients)
    unsigned int cof_n;            // cofactor PIs (2^cof_n copies per iteration)
    unsigned int cof_pos[8];       // their pattern-bit positions (PI - 1), ascending
};

#ifndef ES_MULTI
#define ES_MULTI 0   // 1: cofactor copies (cof_n > 0)
#endif

// pattern index of (word-index bits x, copy 0): zero bits inserted at cof_pos[].
// Runs once per chunk claim; the volatile moves keep the compiler from
// hoisting its masks out of the loop (they would sit in registers the body needs).
__device__ __forceinline__ unsigned long long es_expand(unsigned long long x, const K1Params &p)
{
    unsigned n;
    asm volatile("mov.b32 %0, %1;" : "=r"(n) : "r"(p.cof_n));
#pragma unroll 1
    for (unsigned i = 0; i < n; ++i) {
        unsigned s;
        asm volatile("mov.b32 %0, %1;" : "=r"(s) : "r"(p.cof_pos[i & 7]));
        x = ((x >> s) << (s + 1)) | (x & ((1ull << s) - 1ull));
    }
    return x;
}

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
#if !ES_MULTI
                const unsigned long long first_pattern = (c << p.chunk_log2) << 5;
#else
                const unsigned long long first_pattern = es_expand((c << p.chunk_log2) << 5, p);
#endif
                const unsigned long long b = *(volatile unsigned long long *)p.best;
                // skip rule: every pattern of this chunk (and of every later
                // one) lies above the minimum.  Phase 1 of a non-equivalent
                // search (hit_stop) also stops at the first counterexample and
                // records the lowest slot it left unswept: the host's proof
                // only counts the slots below it as swept
                if (first_pattern > b) {
                    c = ~0ull;
                } else if (b < p.hit_stop) {
                    atomicMin(p.counter + 2, (unsigned)k);
                    c = ~0ull;
                } else {
                    atomicAdd(p.counter + 1, 1u);
                }
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
#if !ES_MULTI
            unsigned out;
            asm volatile("// ES_BODY %0 %1 %2 %3"
                         : "=r"(out) : "r"((unsigned)w), "r"((unsigned)(w >> 32)), "r"(p.one));
            out &= p.valid_mask;
            if (w >= p.total_words) out = 0u;
            const unsigned hit = __ballot_sync(0xffffffffu, out != 0u);
            if (hit) {
                const int l = __ffs(hit) - 1;
                const unsigned ol = __shfl_sync(0xffffffffu, out, l);
                const unsigned long long wl = __shfl_sync(0xffffffffu, w, l);
                // system scope: `best` may be a peer GPU's word mapped over NVLink (CUDA IPC)
                if (lane == 0) atomicMin_system(p.best, (wl << 5) | (unsigned long long)(__ffs(ol) - 1));
            }
#else
            // the body returns the output word of the first failing copy (0: none)
            // and that copy's number; copies are ordered like their pattern indices
            unsigned out, copy;
            asm volatile("// ES_BODY %0 %1 %2 %3 %4"
                         : "=r"(out), "=r"(copy) : "r"((unsigned)w), "r"((unsigned)(w >> 32)), "r"(p.one));
            out &= p.valid_mask;
            if (w >= p.total_words) out = 0u;
            if (__ballot_sync(0xffffffffu, out != 0u)) {
                // rare path: cofactor bits interleave lanes and copies, so take
                // each lane's minimum pattern and reduce over the warp
                unsigned long long cand = ~0ull;
                if (out) {
                    cand = es_expand((w << 5) | (unsigned long long)(__ffs(out) - 1), p);
                    for (unsigned b = 0; b < p.cof_n; ++b)
                        if ((copy >> b) & 1u) cand |= 1ull << p.cof_pos[b];
                }
#pragma unroll
                for (int off = 16; off; off >>= 1) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, cand, off);
                    cand = o < cand ? o : cand;
                }
                // system scope: `best` may be a peer GPU's word mapped over NVLink (CUDA IPC)
                if (lane == 0) atomicMin_system(p.best, cand);
            }
#endif
        }
    }
}
