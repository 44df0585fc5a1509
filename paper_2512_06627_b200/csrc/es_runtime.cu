// es_runtime.cu -- device side of the B200 ES engine: the K2 interpreter
// kernel and the host drivers for es_run / es_run_batch / sessions.
//
// run_exhaustive semantics (cecprove/es.py:252-339) with the minimum-index
// witness of the reference's single-worker sweep (es.py:297-320):
//   * patterns are numbered as in the reference (PI i+1 = bit i of p);
//   * K1 (JIT, k1_skeleton.cu) or K2 (interpreter, below) sweep chunks in
//     increasing order and atomicMin the first failing pattern;
//   * the host runs the sweep in launch slices so the wall budget and the
//     cooperative cancel flag are honoured between slices (es.py:299-309);
//   * patterns_evaluated follows the reference's workers=1 accounting
//     (whole 2^min(n,14)-pattern batches up to and including the hit).
#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "es_core.h"
#include "es_jit.h"
#include "es_k2prog.h"
#include "es_nvtx.h"

namespace es {

void set_error(const std::string &m);

// must match k1_skeleton.cu
struct K1Params {
    unsigned long long *best;
    unsigned int *counter;
    unsigned long long first_chunk;
    unsigned long long n_slots;
    unsigned long long world;
    unsigned long long hit_stop;
    unsigned long long total_words;
    unsigned int chunk_log2;
    unsigned int valid_mask;
    unsigned int one;
    unsigned int cof_n;
    unsigned int cof_pos[8];
};

// ---------------------------------------------------------------------------
// K2: shared-memory interpreter (es_k2prog.cpp builds its programs)
// ---------------------------------------------------------------------------
// Per CTA: the current job's program staged in shared memory (16-byte
// records), then the slot file: slot s of thread t, word k at byte
// s*T*W*4 + t*W*4 + k*4 -- every thread owns its columns, so the gate loop
// needs no barrier, and each access is one W-wide vector (LDS.32/64/128).
// With cofactor copies (es_cofactor.cpp) a job's word index w enumerates the
// non-cofactor PIs only and OUT records fold each copy's output into (first
// failing word, copy); the pattern index inserts the cofactor bits.
struct K2Job {
    const uint4 *code;           // device records, one uint4 per gate / output
    unsigned long long *best;
    unsigned *swept;             // items of this job actually evaluated (not skipped)
    unsigned long long total_words;  // kernel words (cofactor PIs excluded)
    unsigned long long cof_mask;     // bit j: PI j is a cofactor PI
    int n_recs;
    int num_pis;
    unsigned valid_mask;
    int cof_n;
    unsigned char cof_pos[8];        // cofactor pattern bits (PI - 1), ascending
};

struct K2Item {
    unsigned long long w0;
    unsigned n_words;
    int job;
};

// K4 (k4_skeleton.cu, es_sass.cpp): many jobs' straight-line bodies in one
// module behind an indirect branch; the job and parameter layouts mirror the
// skeleton's K4Job / K4Params (items are K2Items)
struct K4JobD {
    unsigned long long total_words;
    unsigned valid_mask;
    unsigned body;
    int cof_n;
    unsigned char cof_pos[8];
};
struct K4ParamsD {
    const K4JobD *jobs;
    const K2Item *items;
    unsigned long long n_items;
    unsigned long long *best;
    unsigned *swept;
    unsigned *counter;
    unsigned one;
};
__constant__ unsigned c_lane_mask[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u,
                                        0xFFFF0000u};

// 32-bit shared-memory accessors (PTX): keeps the slot file in the shared
// window without per-access generic->shared conversion.  All are volatile so
// the compiler keeps program order between the slot loads and stores.
template <int W>
__device__ __forceinline__ void lds(unsigned addr, unsigned (&v)[W]) {
    if constexpr (W == 1) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[0]) : "r"(addr));
    if constexpr (W == 2) asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(addr));
    if constexpr (W == 4)
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
}
template <int W>
__device__ __forceinline__ void sts(unsigned addr, const unsigned (&v)[W]) {
    if constexpr (W == 1) asm volatile("st.shared.u32 [%0], %1;" :: "r"(addr), "r"(v[0]) : "memory");
    if constexpr (W == 2) asm volatile("st.shared.v2.u32 [%0], {%1, %2};" :: "r"(addr), "r"(v[0]), "r"(v[1]) : "memory");
    if constexpr (W == 4)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};"
                     :: "r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
}
__device__ __forceinline__ uint4 lds_rec(unsigned addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
    return r;
}

// pattern index of kernel word bits x with zero bits inserted at cof_pos[]
__device__ __forceinline__ unsigned long long k2_expand(unsigned long long x, const K2Job &job) {
    for (int i = 0; i < job.cof_n; ++i) {
        const unsigned s = job.cof_pos[i];
        x = ((x >> s) << (s + 1)) | (x & ((1ull << s) - 1ull));
    }
    return x;
}

template <int W>
__global__ void __launch_bounds__(128) es_k2(const K2Job *__restrict__ jobs,
                                             const K2Item *__restrict__ items,
                                             unsigned long long item_begin,
                                             unsigned long long item_end, unsigned *counter,
                                             int smem_bytes) {
    // dynamic shared memory: the slot file from the bottom, the current job's
    // records (plus one past-end record for the prefetch) at the top, so a job
    // needs slots * 512 * W + (records + 1) * 16 bytes of its own, not the
    // group's largest slot file plus its longest program
    extern __shared__ __align__(16) uint4 smem[];
    __shared__ unsigned long long s_item;
    const unsigned T = blockDim.x, t = threadIdx.x, lane = t & 31u;
    const unsigned smem_addr = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned base = smem_addr + t * W * 4;
    unsigned prog_addr = smem_addr;
    const unsigned long long kStop = ~0ull, kSkip = ~0ull - 1;
    int cur_job = -1;
    for (;;) {
        if (t == 0) {
            unsigned long long k = item_begin + atomicAdd(counter, 1u);
            if (k >= item_end) {
                k = kStop;
            } else {
                const K2Item it = items[k];
                const K2Job &jb = jobs[it.job];
                if (k2_expand(it.w0 << 5, jb) > *(volatile unsigned long long *)jb.best) k = kSkip;
                else atomicAdd(jb.swept, 1u);
            }
            s_item = k;
        }
        __syncthreads();
        const unsigned long long k = s_item;
        if (k == kStop) break;
        if (k == kSkip) { __syncthreads(); continue; }
        const K2Item it = items[k];
        const K2Job job = jobs[it.job];
        const int rec0 = smem_bytes / 16 - (job.n_recs + 1);
        prog_addr = smem_addr + 16u * (unsigned)rec0;
        if (it.job != cur_job) {  // stage the program records (uniform branch)
            const uint4 *src = reinterpret_cast<const uint4 *>(job.code);
            for (int q = t; q < job.n_recs; q += T) smem[rec0 + q] = __ldg(&src[q]);
            cur_job = it.job;
        }
        __syncthreads();
        for (unsigned wb = 0; wb < it.n_words; wb += T * W) {
            const unsigned long long w = it.w0 + wb + (unsigned long long)t * W;
            // PI words into slots 0..n-1: lane PIs are constants, cofactor PIs
            // are folded into the program, the rest are bits of w
            {
                int bit = 0;
                for (int j = 0; j < job.num_pis; ++j) {
                    if (j >= 5 && ((job.cof_mask >> (j + 1)) & 1ull)) continue;
                    unsigned v[W];
#pragma unroll
                    for (int q = 0; q < W; ++q)
                        v[q] = j < 5 ? c_lane_mask[j] : ((((w + q) >> bit) & 1ull) ? ~0u : 0u);
                    if (j >= 5) ++bit;
                    sts<W>(base + (unsigned)j * T * W * 4, v);
                }
            }
            unsigned acc[W], fw[W], fc[W];
#pragma unroll
            for (int q = 0; q < W; ++q) { acc[q] = 0; fw[q] = 0; fc[q] = 0; }
            // Records {off_a, off_b, off_d, ctl}.  Gates: operand A is the
            // accumulator or is loaded into it, B is a slot, the result stays
            // in the accumulator and is stored only if read later.  OUT: fold
            // the copy's output into (first failing word, copy) per word.
            uint4 r0 = lds_rec(prog_addr);
            // Unrolled 8x; this file is compiled with ptxas
            // --register-usage-level=10 (build.py): config 4 20.0 ms (at the
            // default level 5: 1x 26.4 ms, ptxas's own 2x 24.5, 8x 22.6).
#pragma unroll 8
            for (int i = 0; i < job.n_recs; ++i) {
                const uint4 c0 = r0;
                r0 = lds_rec(prog_addr + 16u * (unsigned)(i + 1));  // next record (past-end reads harmless)
                const unsigned ma = (unsigned)((int)c0.w >> 31);  // NEG_A mirrored in bit 31
                if (c0.w & K2_OUT) {
                    unsigned v[W];
                    if (c0.w & K2_A_ACC) {
#pragma unroll
                        for (int q = 0; q < W; ++q) v[q] = acc[q];
                    } else if (c0.w & K2_CONST) {
#pragma unroll
                        for (int q = 0; q < W; ++q) v[q] = 0u;
                    } else {
                        lds<W>(base + c0.x, v);
                    }
                    const unsigned copy = (c0.w >> 16) & 0x3FFFu;
#pragma unroll
                    for (int q = 0; q < W; ++q) {
                        const bool first = fw[q] == 0u;
                        fw[q] = first ? (v[q] ^ ma) : fw[q];
                        fc[q] = first ? copy : fc[q];
                    }
                    continue;
                }
                unsigned b[W];
                if (!(c0.w & K2_A_ACC)) lds<W>(base + c0.x, acc);
                lds<W>(base + c0.y, b);
                if (c0.w & K2_XOR) {
#pragma unroll
                    for (int q = 0; q < W; ++q) acc[q] = acc[q] ^ b[q] ^ ma;
                } else {
                    const unsigned mb = (unsigned)((int)(c0.w << 1) >> 31);  // NEG_B in bit 30
#pragma unroll
                    for (int q = 0; q < W; ++q) acc[q] = (acc[q] ^ ma) & (b[q] ^ mb);
                }
                if (c0.w & K2_STORE) sts<W>(base + c0.z, acc);
            }
            unsigned any = 0;
#pragma unroll
            for (int q = 0; q < W; ++q) {
                unsigned o = fw[q] & job.valid_mask;
                if (w + q >= job.total_words || wb + t * W + q >= it.n_words) o = 0;
                fw[q] = o;
                any |= o;
            }
            if (__ballot_sync(0xffffffffu, any != 0u)) {
                // rare path: each lane's minimum pattern (cofactor bits
                // interleave words and copies), then the warp minimum
                unsigned long long cand = ~0ull;
#pragma unroll
                for (int q = 0; q < W; ++q) {
                    if (!fw[q]) continue;
                    unsigned long long pat = k2_expand(((w + q) << 5) | (unsigned long long)(__ffs(fw[q]) - 1), job);
                    for (int b2 = 0; b2 < job.cof_n; ++b2)
                        if ((fc[q] >> b2) & 1u) pat |= 1ull << job.cof_pos[b2];
                    cand = pat < cand ? pat : cand;
                }
#pragma unroll
                for (int off = 16; off; off >>= 1) {
                    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, cand, off);
                    cand = o2 < cand ? o2 : cand;
                }
                if (lane == 0) atomicMin(job.best, cand);
            }
        }
    }
}

// K2, L lanes (multi-lane programs, es_k2prog.cpp emit_k2_lanes): every
// step is L records -- L independent gates with one accumulator per lane,
// or up to L OUT records -- so a warp has L dependency chains to issue from
// (the one-lane kernel is latency-bound at 8 warps per SM: stall_wait 2.2
// per issue).  Every lane's operands are loaded before any result of the step
// is stored; slot num_pis holds zero (a NOP lane is acc & ~0 over it).
#ifndef ES_K2D_UNROLL
#define ES_K2D_UNROLL 2
#endif
template <int W, int L>
__global__ void __launch_bounds__(128) es_k2d(const K2Job *__restrict__ jobs,
                                              const K2Item *__restrict__ items,
                                              unsigned long long item_begin,
                                              unsigned long long item_end, unsigned *counter,
                                              int smem_bytes) {
    extern __shared__ __align__(16) uint4 smem[];
    __shared__ unsigned long long s_item;
    const unsigned T = blockDim.x, t = threadIdx.x, lane = t & 31u;
    const unsigned smem_addr = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned base = smem_addr + t * W * 4;
    unsigned prog_addr = smem_addr;
    const unsigned long long kStop = ~0ull, kSkip = ~0ull - 1;
    int cur_job = -1;
    for (;;) {
        if (t == 0) {
            unsigned long long k = item_begin + atomicAdd(counter, 1u);
            if (k >= item_end) {
                k = kStop;
            } else {
                const K2Item it = items[k];
                const K2Job &jb = jobs[it.job];
                if (k2_expand(it.w0 << 5, jb) > *(volatile unsigned long long *)jb.best) k = kSkip;
                else atomicAdd(jb.swept, 1u);
            }
            s_item = k;
        }
        __syncthreads();
        const unsigned long long k = s_item;
        if (k == kStop) break;
        if (k == kSkip) { __syncthreads(); continue; }
        const K2Item it = items[k];
        const K2Job job = jobs[it.job];
        // records, then room for one step's prefetch past the end
        const int rec0 = smem_bytes / 16 - (job.n_recs + kK2PadRecords);
        prog_addr = smem_addr + 16u * (unsigned)rec0;
        if (it.job != cur_job) {
            const uint4 *src = reinterpret_cast<const uint4 *>(job.code);
            for (int q = t; q < job.n_recs; q += T) smem[rec0 + q] = __ldg(&src[q]);
            cur_job = it.job;
        }
        __syncthreads();
        const int n_steps = job.n_recs / L;
        for (unsigned wb = 0; wb < it.n_words; wb += T * W) {
            const unsigned long long w = it.w0 + wb + (unsigned long long)t * W;
            {
                int bit = 0;
                for (int j = 0; j < job.num_pis; ++j) {
                    if (j >= 5 && ((job.cof_mask >> (j + 1)) & 1ull)) continue;
                    unsigned v[W];
#pragma unroll
                    for (int q = 0; q < W; ++q)
                        v[q] = j < 5 ? c_lane_mask[j] : ((((w + q) >> bit) & 1ull) ? ~0u : 0u);
                    if (j >= 5) ++bit;
                    sts<W>(base + (unsigned)j * T * W * 4, v);
                }
                unsigned z[W];
#pragma unroll
                for (int q = 0; q < W; ++q) z[q] = 0u;
                sts<W>(base + (unsigned)job.num_pis * T * W * 4, z);  // the NOP lanes' zero slot
            }
            unsigned acc[L][W], b[L][W], fw[W], fc[W];
#pragma unroll
            for (int h = 0; h < L; ++h)
#pragma unroll
                for (int q = 0; q < W; ++q) acc[h][q] = 0;
#pragma unroll
            for (int q = 0; q < W; ++q) { fw[q] = 0; fc[q] = 0; }
            // the current step's records c[], the next step's nx[], and c's
            // decoded operand addresses and masks; each step ends by decoding
            // the next one inside its own basic block, so the decode overlaps
            // the step's logic instead of heading the next block
            uint4 c[L], nx[L];
            unsigned pa[L], pb[L], pd[L], ma[L], mb[L], ms[L];
#pragma unroll
            for (int h = 0; h < L; ++h) {
                c[h] = lds_rec(prog_addr + 16u * h);
                nx[h] = lds_rec(prog_addr + 16u * (L + h));
            }
            // masks from the msb of ctl bytes 3 / 2 / 1 (NEG_A, NEG_B, XOR;
            // packed by k2_group_prepare), one PRMT each
            auto decode = [&]() {
#pragma unroll
                for (int h = 0; h < L; ++h) {
                    pa[h] = base + c[h].x;
                    pb[h] = base + c[h].y;
                    pd[h] = base + c[h].z;
                    asm("prmt.b32 %0, %1, 0, 0xBBBB;" : "=r"(ma[h]) : "r"(c[h].w));
                    asm("prmt.b32 %0, %1, 0, 0xAAAA;" : "=r"(mb[h]) : "r"(c[h].w));
                    asm("prmt.b32 %0, %1, 0, 0x9999;" : "=r"(ms[h]) : "r"(c[h].w));
                }
            };
            decode();
#pragma unroll 2
            for (int i = 0; i < n_steps; ++i) {
                // step i+2's records (past-end reads harmless: kK2PadRecords)
                auto advance = [&]() {
#pragma unroll
                    for (int h = 0; h < L; ++h) {
                        c[h] = nx[h];
                        nx[h] = lds_rec(prog_addr + 16u * (unsigned)(L * (i + 2) + h));
                    }
                    decode();
                };
                if (c[0].w & K2_OUT) {  // OUT step: fold in record (= copy) order
#pragma unroll
                    for (int h = 0; h < L; ++h) {
                        if (!(c[h].w & K2_OUT)) continue;
                        unsigned v[W];
                        if (c[h].w & K2_A_ACC) {
                            const unsigned ln = (c[h].w >> K2_OUT_LANE_SHIFT) & 3u;
#pragma unroll
                            for (int q = 0; q < W; ++q) {
                                unsigned x = acc[0][q];
#pragma unroll
                                for (int g = 1; g < L; ++g) x = ln == (unsigned)g ? acc[g][q] : x;
                                v[q] = x;
                            }
                        } else if (c[h].w & K2_CONST) {
#pragma unroll
                            for (int q = 0; q < W; ++q) v[q] = 0u;
                        } else {
                            lds<W>(pa[h], v);
                        }
                        const unsigned copy = (c[h].w >> 16) & 0x3FFFu;
#pragma unroll
                        for (int q = 0; q < W; ++q) {
                            const bool first = fw[q] == 0u;
                            fw[q] = first ? (v[q] ^ ma[h]) : fw[q];
                            fc[q] = first ? copy : fc[q];
                        }
                    }
                    advance();
                    continue;
                }
                // every lane's loads first (A straight into its accumulator)
#pragma unroll
                for (int h = 0; h < L; ++h) {
                    if (!(c[h].w & K2_A_ACC)) lds<W>(pa[h], acc[h]);
                    lds<W>(pb[h], b[h]);
                }
                // u = A ^ ma, t = B ^ mb, result = s ? u ^ t : u & t
#pragma unroll
                for (int h = 0; h < L; ++h)
#pragma unroll
                    for (int q = 0; q < W; ++q) {
                        const unsigned u = acc[h][q] ^ ma[h], tt = b[h][q] ^ mb[h];
                        unsigned r;  // one LOP3 (0x68 over u, t, s)
                        asm("lop3.b32 %0, %1, %2, %3, 0x68;" : "=r"(r) : "r"(u), "r"(tt), "r"(ms[h]));
                        acc[h][q] = r;
                    }
#pragma unroll
                for (int h = 0; h < L; ++h)
                    sts<W>(pd[h], acc[h]);  // (unread results go to the program's dummy slot)
                advance();
            }
            unsigned any = 0;
#pragma unroll
            for (int q = 0; q < W; ++q) {
                unsigned o = fw[q] & job.valid_mask;
                if (w + q >= job.total_words || wb + t * W + q >= it.n_words) o = 0;
                fw[q] = o;
                any |= o;
            }
            if (__ballot_sync(0xffffffffu, any != 0u)) {
                unsigned long long cand = ~0ull;
#pragma unroll
                for (int q = 0; q < W; ++q) {
                    if (!fw[q]) continue;
                    unsigned long long pat = k2_expand(((w + q) << 5) | (unsigned long long)(__ffs(fw[q]) - 1), job);
                    for (int b2 = 0; b2 < job.cof_n; ++b2)
                        if ((fc[q] >> b2) & 1u) pat |= 1ull << job.cof_pos[b2];
                    cand = pat < cand ? pat : cand;
                }
#pragma unroll
                for (int off = 16; off; off >>= 1) {
                    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, cand, off);
                    cand = o2 < cand ? o2 : cand;
                }
                if (lane == 0) atomicMin(job.best, cand);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// ALU-pipe peak microbenchmark: 8 independent LOP3 chains per thread, enough
// warps to saturate every SMSP.  Gives the measured roofline denominator for
// bit-parallel simulation (lane-LOP3/s); MEASURED_PEAKS.json has no integer
// figure.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) es_alu_peak_kernel(unsigned *sink, int iters, unsigned seed) {
    unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
    unsigned a4 = a0 * 11u, a5 = a0 * 13u, a6 = a0 * 17u, a7 = a0 * 19u;
#define ES_L3(d, x, y, z, lut) asm volatile("lop3.b32 %0, %1, %2, %3, " #lut ";" : "=r"(d) : "r"(x), "r"(y), "r"(z))
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ES_L3(a0, a0, a1, a2, 0x96); ES_L3(a1, a1, a2, a3, 0xE8);
            ES_L3(a2, a2, a3, a4, 0x96); ES_L3(a3, a3, a4, a5, 0xE8);
            ES_L3(a4, a4, a5, a6, 0x96); ES_L3(a5, a5, a6, a7, 0xE8);
            ES_L3(a6, a6, a7, a0, 0x96); ES_L3(a7, a7, a0, a1, 0xE8);
        }
    }
#undef ES_L3
    const unsigned r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
    if (r == 0x9E3779B9u) sink[0] = r;
}

int alu_peak(int dev, double *lane_ops_per_s, double *ms_out);

// FMA-pipe integer peak: 8 independent IMAD chains per thread (the K1 body's
// x*S+T LUTs and coefficients run there).  Measured on the B200: 1.84e13
// lane-IMAD/s, the same as the ALU pipe's LOP3 peak.  The multiplier is
// opaque (from the seed) so ptxas cannot strength-reduce the chains.
__global__ void __launch_bounds__(256) es_imad_peak_kernel(unsigned *sink, int iters, unsigned seed) {
    unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
    unsigned a4 = a0 * 11u, a5 = a0 * 13u, a6 = a0 * 17u, a7 = a0 * 19u;
    const unsigned m = seed | 0x10001u;
#define ES_MAD(d, x, y) asm volatile("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(m), "r"(y))
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ES_MAD(a0, a0, a1); ES_MAD(a1, a1, a2); ES_MAD(a2, a2, a3); ES_MAD(a3, a3, a4);
            ES_MAD(a4, a4, a5); ES_MAD(a5, a5, a6); ES_MAD(a6, a6, a7); ES_MAD(a7, a7, a0);
        }
    }
#undef ES_MAD
    const unsigned r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
    if (r == 0x9E3779B9u) sink[0] = r;
}

int fma_peak(int dev, double *lane_ops_per_s, double *ms_out);

// *w = min(*w, *v): folds the other devices' minimum into a device-local word
// (multi-GPU sweep without peer access)
__global__ void es_word_min_kernel(unsigned long long *w, const unsigned long long *v) { atomicMin(w, *v); }

// Shared-memory load bandwidth microbenchmark (the K2 interpreter's slot file
// is a shared-memory bound): conflict-free 16-byte loads, 8
// independent per thread per iteration, over a 16 KB tile per CTA.
__global__ void __launch_bounds__(256) es_smem_peak_kernel(unsigned *sink, int iters) {
    __shared__ __align__(16) uint4 tile[1024];
    for (int q = threadIdx.x; q < 1024; q += blockDim.x) tile[q] = make_uint4(q, q * 3u, q * 5u, q * 7u);
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(tile);
    unsigned x = 0, y = 0, z = 0, w = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const unsigned addr = base + 16u * ((threadIdx.x + 128u * k + (unsigned)i) & 1023u);
            unsigned a, b, c, d;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
            x ^= a; y ^= b; z ^= c; w ^= d;
        }
    }
    if ((x ^ y ^ z ^ w) == 0x9E3779B9u) sink[0] = x;
}

// ---------------------------------------------------------------------------
// per-device contexts, leased for the duration of one call
// ---------------------------------------------------------------------------
namespace {

struct Ctx {
    int dev = -1;
    int sms = 0;
    cudaStream_t stream = nullptr;
    unsigned long long *d_best = nullptr;  // [0] best
    unsigned *d_counter = nullptr;         // [2] per in-flight slice
    unsigned long long *h_pin = nullptr;   // [4]
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr, ev_slice[2] = {nullptr, nullptr};
    // concurrent K2 launch groups [0, 3) and K4 module launches [3, 7)
    cudaStream_t side[7] = {};
    cudaEvent_t ev_side[7] = {};
    uint4 *h_stage = nullptr;  // pinned staging of K2 program records (grown on demand)
    size_t stage_cap = 0;      // in records
};

// Every call leases one context per device it runs on (a stream, the slice
// words, events) and returns it when it ends, so concurrent callers (the
// scheduler races ES against SAT/BDD on several host threads, and a
// multi-GPU sweep drives each device from its own host thread) never share
// a stream, while a context outlives the thread that made it.
std::mutex g_ctx_mu;
std::vector<Ctx *> g_ctx_all, g_ctx_free;

int cuda_fail(cudaError_t e, const char *what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return ES_E_CUDA;
}

#define CK(call)                                          \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

int make_ctx(int dev, Ctx *c) {
    c->dev = dev;
    CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev));
    {
        // keep freed stream-ordered allocations in the pool: the K2 / K3 drivers
        // allocate per call, and a pool that trims at every synchronize goes
        // back to the driver each time (measured: 0.5 -> 11 ms per small K2 run
        // once another process had used the GPU)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&c->d_best, 64));
    CK(cudaMalloc(&c->d_counter, 64));
    CK(cudaMallocHost(&c->h_pin, 64));
    CK(cudaEventCreate(&c->ev_start));
    CK(cudaEventCreate(&c->ev_stop));
    CK(cudaEventCreateWithFlags(&c->ev_slice[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_slice[1], cudaEventDisableTiming));
    for (int q = 0; q < 7; ++q) {
        CK(cudaStreamCreateWithFlags(&c->side[q], cudaStreamNonBlocking));
        CK(cudaEventCreate(&c->ev_side[q]));
    }
    return ES_OK;
}

int check_device(int dev) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        set_error("no CUDA device visible");
        return ES_E_NO_DEVICE;
    }
    if (dev < 0 || dev >= n) {
        set_error("device ordinal " + std::to_string(dev) + " out of range (" + std::to_string(n) + " visible)");
        return ES_E_BAD_ARG;
    }
    return ES_OK;
}

struct CtxLease {
    Ctx *c = nullptr;
    CtxLease() = default;
    CtxLease(const CtxLease &) = delete;
    CtxLease &operator=(const CtxLease &) = delete;
    int acquire(int dev) {
        int rc = check_device(dev);
        if (rc != ES_OK) return rc;
        CK(cudaSetDevice(dev));
        {
            std::lock_guard<std::mutex> lk(g_ctx_mu);
            for (size_t i = 0; i < g_ctx_free.size(); ++i)
                if (g_ctx_free[i]->dev == dev) {
                    c = g_ctx_free[i];
                    g_ctx_free.erase(g_ctx_free.begin() + (long)i);
                    return ES_OK;
                }
        }
        Ctx *n = new Ctx();
        rc = make_ctx(dev, n);
        if (rc != ES_OK) { delete n; return rc; }  // (partially created CUDA objects leak; rare)
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        g_ctx_all.push_back(n);
        c = n;
        return ES_OK;
    }
    ~CtxLease() {
        if (!c) return;
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        g_ctx_free.push_back(c);
    }
};

inline uint64_t ref_patterns_for_hit(uint64_t idx, int P) {
    const int b = std::min(P, 14);  // reference batch = 2^min(n,14) patterns
    return ((idx >> b) + 1) << b;
}

bool stop_requested(const es_run_opts &o, double deadline, int *reason) {
    if (deadline >= 0 && now_ms() >= deadline) { *reason = ES_REASON_TIMEOUT; return true; }
    if (o.cancel_flag && *o.cancel_flag) { *reason = ES_REASON_CANCELLED; return true; }
    return false;
}

// words per chunk: small enough for a balanced tail, large enough to amortise
// the claim (one atomic + two barriers per chunk)
int pick_chunk_log2(uint64_t total_words, int threads, int resident_ctas) {
    const int tw = total_words ? 63 - __builtin_clzll(total_words) : 0;
    int lg = 0;
    while ((1 << lg) < threads) ++lg;
    // aim for >= 32 chunks per resident CTA over the whole space (a rank of
    // an 8-GPU shard still gets ~4: a small tail), cap at 2^13 words
    int per_cta = 32;  // measured: full mult16 +0.5 %, its 1/8 shard -11 % vs 16
    if (const char *e = getenv("ES_CHUNKS_PER_CTA")) per_cta = std::max(1, atoi(e));
    int want = tw - (int)std::ceil(std::log2(std::max(1, resident_ctas * per_cta)));
    want = std::min(want, 13);
    return std::max(lg, want);
}

}  // namespace

// ---------------------------------------------------------------------------
// K1 driver
// ---------------------------------------------------------------------------
struct K1Plan {
    JitKernel *jk = nullptr;
    int threads = 256;     // CTA size
    size_t smem = 0;       // dynamic shared bytes (K1T)
    int chunk_log2 = 8;
    uint64_t total_words = 1;  // of the kernel's word index (cofactor PIs excluded)
    uint64_t n_chunks = 1;
    int grid = 1;
    uint32_t valid = 0;
    int cof_n = 0;             // cofactor PIs: 2^cof_n words per iteration
    unsigned cof_pos[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // pattern index of the first pattern of chunk c (copy 0): the kernel's
    // es_expand on the host; monotone in c
    uint64_t first_pattern(uint64_t c) const {
        uint64_t x = (c << chunk_log2) << 5;
        for (int i = 0; i < cof_n; ++i) {
            const unsigned sh = cof_pos[i];
            x = ((x >> sh) << (sh + 1)) | (x & ((1ull << sh) - 1ull));
        }
        return x;
    }
    uint64_t patterns_per_chunk() const { return 1ull << (chunk_log2 + 5 + cof_n); }
};

int k1_prepare(const LutNet &net, int threads, int sms, K1Plan *pl, double *jit_ms,
               JitKernel *cached = nullptr, int opt = 3, int n_dev = 1) {
    std::string err;
    if (cached) {
        pl->jk = cached;
        *jit_ms = 0.0;
    } else {
        int rc = jit_get(net, threads, &pl->jk, jit_ms, &err, opt);
        if (rc != ES_OK) { set_error(err); return rc; }
    }
    pl->threads = pl->jk->block;
    pl->smem = (size_t)pl->jk->region_bytes;  // split build: the slot file
    const int P = net.num_pis;
    pl->cof_n = (int)net.cof_pis.size();
    if (pl->cof_n > kMaxCofactorPis || (pl->cof_n > 0 && P - 5 - pl->cof_n < 0)) { set_error("bad cofactor set"); return ES_E_BAD_ARG; }
    for (int i = 0; i < pl->cof_n; ++i) pl->cof_pos[i] = (unsigned)(net.cof_pis[i] - 1);
    pl->total_words = 1ull << std::max(P - 5 - pl->cof_n, 0);
    int nb = 0;
    if (getenv("ES_VERBOSE")) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, (const void *)pl->jk->kernel);
        fprintf(stderr, "[es] K1 kernel: regs %d local %zu B static smem %zu B max threads %d, dynamic smem %zu B, parts %d\n",
                fa.numRegs, (size_t)fa.localSizeBytes, (size_t)fa.sharedSizeBytes, fa.maxThreadsPerBlock, pl->smem,
                pl->jk->parts);
    }
    if (pl->smem > 0)  // the skeleton's static shared memory counts against the 48 KB default too
        CK(cudaFuncSetAttribute((const void *)pl->jk->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)pl->jk->kernel, pl->threads, pl->smem));
    nb = std::max(nb, 1);
    const int min_words = pl->threads;
    // chunk size for the whole job: n_dev GPUs' resident CTAs share the chunks
    pl->chunk_log2 = pick_chunk_log2(pl->total_words, min_words, sms * nb * std::max(1, n_dev));
    pl->n_chunks = std::max<uint64_t>(1, pl->total_words >> pl->chunk_log2);
    pl->grid = (int)std::min<uint64_t>(pl->n_chunks, (uint64_t)sms * nb);
    pl->valid = lane_valid_mask(P);
    return ES_OK;
}

// counter: three words, [0] claims, [1] chunks swept (zeroed here) and [2]
// the lowest slot a hit_stop launch left unswept (set to ~0 here)
int k1_launch(const K1Plan &pl, cudaStream_t st, unsigned long long *best, unsigned *counter,
              uint64_t first_chunk, uint64_t n_slots, uint64_t world, uint64_t hit_stop = 0) {
    K1Params kp;
    kp.best = best;
    kp.counter = counter;
    kp.first_chunk = first_chunk;
    kp.n_slots = n_slots;
    kp.world = world;
    kp.hit_stop = hit_stop;
    kp.total_words = pl.total_words;
    kp.chunk_log2 = (unsigned)pl.chunk_log2;
    kp.valid_mask = pl.valid;
    kp.one = 1u;
    kp.cof_n = (unsigned)pl.cof_n;
    for (int i = 0; i < 8; ++i) kp.cof_pos[i] = pl.cof_pos[i];
    CK(cudaMemsetAsync(counter, 0, 2 * sizeof(unsigned), st));
    CK(cudaMemsetAsync(counter + 2, 0xFF, sizeof(unsigned), st));
    void *args[] = {&kp};
    const int grid = (int)std::min<uint64_t>((uint64_t)pl.grid, std::max<uint64_t>(n_slots, 1));
    CK(cudaLaunchKernel((const void *)pl.jk->kernel, dim3(grid), dim3(pl.threads), args, pl.smem, st));
    return ES_OK;
}

// Default CTA size: 128 for one word per iteration (165 registers: 3 CTAs
// per SM), 256 with cofactor copies (255 registers; measured 10-15% faster).
static int k1_threads(const es_run_opts &o, int cofactor_pis = 0) {
    return o.block_threads > 0 ? o.block_threads : cofactor_pis > 0 ? 256 : 128;
}
static int k1_slot(int threads) { return threads == 128 ? 0 : threads == 256 ? 1 : 2; }

// The devices of one run: es_run_opts.devices[0..n_devices) when given (the
// same ordinal may repeat: several host threads then share one GPU), else
// es_run_opts.device.
static std::vector<int> run_devices(const es_run_opts &o) {
    std::vector<int> d;
    if (o.n_devices > 0 && o.devices)
        for (int i = 0; i < o.n_devices; ++i) d.push_back(o.devices[i]);
    if (d.empty()) d.push_back(o.device);
    return d;
}

// ---------------------------------------------------------------------------
// Multi-device K1 sweep.  Global chunks [begin, n_chunks) are
// dealt round-robin: device d sweeps begin + d + k*n.  Every device is driven
// by its own host thread in launch slices, and all kernels atomicMin into ONE
// minimum word in device 0's HBM, reached by the other GPUs as peer memory
// over NVLink/NVSwitch (system-scope atomics): a counterexample found on any
// GPU stops every GPU at its next chunk claim, with no collective on the data
// path.  Without peer access each device keeps its own word and the host
// threads combine them between slices.  The swept prefix is tracked per
// device, so the minimum-index proof (best below the first pattern of the
// first unswept chunk) holds across devices.
// ---------------------------------------------------------------------------
struct SweepOut {
    uint64_t best = 0;        // minimum failing pattern found (init_best if none)
    uint64_t prefix = 0;      // global chunks [0, prefix) fully swept
    uint64_t swept = 0;       // chunks swept (all devices, completed launches)
    bool stopped = false;     // budget / cancel
    int reason = 0;
    double device_ms = 0;     // max over devices of the slices' CUDA-event time
    int launches = 0;
};

static int sweep_k1(const K1Plan &pl, int G, const es_run_opts &o, const std::vector<Ctx *> &cs,
                    double deadline, uint64_t begin, uint64_t init_best, uint64_t hit_stop,
                    SweepOut *res, uint64_t end = ~0ull) {
    const int n = (int)cs.size();
    const uint64_t N = std::min(end, pl.n_chunks);  // this sweep covers global chunks [begin, N)
    // the shared word: device 0's, if every other device can reach it
    bool shared = true;
    for (int d = 1; d < n && shared; ++d) {
        if (cs[d]->dev == cs[0]->dev) continue;
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, cs[d]->dev, cs[0]->dev) != cudaSuccess || !can) { shared = false; break; }
        CK(cudaSetDevice(cs[d]->dev));
        const cudaError_t e = cudaDeviceEnablePeerAccess(cs[0]->dev, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) { cudaGetLastError(); shared = false; }
    }
    std::vector<unsigned long long *> word(n);
    for (int d = 0; d < n; ++d) word[d] = shared ? cs[0]->d_best : cs[d]->d_best;
    for (int d = 0; d < n; ++d) {
        if (d > 0 && shared) continue;
        CK(cudaSetDevice(cs[d]->dev));
        cs[d]->h_pin[0] = init_best;
        CK(cudaMemcpyAsync(cs[d]->d_best, cs[d]->h_pin, 8, cudaMemcpyHostToDevice, cs[d]->stream));
        // armed before any device launches: one device's launches follow the
        // copy in stream order; other devices' streams need the host to wait
        if (n > 1) CK(cudaStreamSynchronize(cs[d]->stream));
    }
    // slice size (in this device's chunk slots) from a conservative rate estimate
    const bool sliced = deadline >= 0 || o.cancel_flag != nullptr;
    const double slice_ms = o.slice_ms > 0 ? o.slice_ms : 20.0;
    const double est_rate = 2.0e14;  // gate-patterns/s per GPU, deliberately low
    const double chunk_ms = 1e3 * (double)std::max(G, 1) * (double)pl.patterns_per_chunk() / est_rate;
    uint64_t per_slice_all = sliced ? (uint64_t)std::max(1.0, slice_ms / chunk_ms) : N;
    per_slice_all = std::max<uint64_t>(per_slice_all, (uint64_t)pl.grid);

    std::vector<std::atomic<uint64_t>> progress(n);  // per device: slots swept (prefix of its class)
    std::vector<uint64_t> slots(n, 0);
    for (int d = 0; d < n; ++d) {
        slots[d] = N > begin + d ? (N - begin - d + n - 1) / n : 0;
        progress[d].store(0);
    }
    std::atomic<uint64_t> best{init_best};
    std::atomic<bool> done{false};
    std::atomic<int> stop_reason{0}, err{ES_OK}, launches{0};
    std::atomic<uint64_t> swept{0};
    std::mutex err_mu;
    std::string err_msg;
    std::vector<double> dev_ms(n, 0.0);
    auto prefix = [&]() {  // global chunks [0, p) all swept
        uint64_t p = N;
        for (int d = 0; d < n; ++d) {
            const uint64_t pr = progress[d].load();
            if (pr < slots[d]) p = std::min(p, begin + pr * n + d);
        }
        return p;
    };
    auto lower = [&](uint64_t v) {
        uint64_t cur = best.load();
        while (v < cur && !best.compare_exchange_weak(cur, v)) {}
    };
    auto settled = [&]() {  // nothing below `best` is left unswept, or phase 1 saw a hit
        const uint64_t b = best.load();
        if (b < hit_stop) return true;
        const uint64_t p = prefix();
        return p >= N || b < pl.first_pattern(p);
    };
    auto worker = [&](int d) {
        Ctx *c = cs[d];
        auto fail = [&](int rc) {
            std::lock_guard<std::mutex> lk(err_mu);
            if (err.load() == ES_OK) { err.store(rc); err_msg = es_last_error(); }
            done.store(true);
        };
        if (cudaSetDevice(c->dev) != cudaSuccess) { fail(cuda_fail(cudaGetLastError(), "cudaSetDevice")); return; }
        const uint64_t per_slice = std::max<uint64_t>(1, per_slice_all);
        std::vector<uint64_t> slice_end;
        int my = 0;
        if (cudaEventRecord(c->ev_start, c->stream) != cudaSuccess) { fail(cuda_fail(cudaGetLastError(), "event")); return; }
        // per slice q: h_cnt[4q + 1] chunks swept, h_cnt[4q + 2] first slot left by hit_stop
        unsigned *h_cnt = reinterpret_cast<unsigned *>(c->h_pin + 4);
        std::vector<uint64_t> slice_begin;
        auto harvest = [&](int q, uint64_t b0, uint64_t end) {  // slice q's copies have landed
            lower(c->h_pin[1 + q]);
            swept.fetch_add(h_cnt[4 * q + 1]);
            // every slot below the first one hit_stop skipped was swept (the
            // claims are in slot order); later ones only by chance
            const uint64_t cut = h_cnt[4 * q + 2] == ~0u ? end : std::min<uint64_t>(end, b0 + h_cnt[4 * q + 2]);
            if (cut > progress[d].load()) progress[d].store(cut);
            if (settled()) done.store(true);
        };
        for (uint64_t b = 0; b < slots[d] && !done.load(); b += per_slice) {
            int reason = 0;
            if (stop_requested(o, deadline, &reason)) {
                int z = 0;
                stop_reason.compare_exchange_strong(z, reason);
                done.store(true);
                break;
            }
            const uint64_t ns = std::min(per_slice, slots[d] - b);
            const int s = my & 1;
            if (!shared) {  // fold the other devices' finds into this device's word first
                const uint64_t g = best.load();
                if (g < init_best) {
                    c->h_pin[3] = g;
                    if (cudaMemcpyAsync(c->d_best + 1, c->h_pin + 3, 8, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
                        fail(cuda_fail(cudaGetLastError(), "cudaMemcpyAsync")); return;
                    }
                    es_word_min_kernel<<<1, 1, 0, c->stream>>>(c->d_best, c->d_best + 1);
                }
            }
            int rc = k1_launch(pl, c->stream, word[d], c->d_counter + 4 * s, begin + d + b * n, ns,
                               (uint64_t)n, hit_stop);
            if (rc != ES_OK) { fail(rc); return; }
            if (cudaMemcpyAsync(c->h_pin + 1 + s, word[d], 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                cudaMemcpyAsync(h_cnt + 4 * s, c->d_counter + 4 * s, 12, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                cudaEventRecord(c->ev_slice[s], c->stream) != cudaSuccess) {
                fail(cuda_fail(cudaGetLastError(), "slice bookkeeping")); return;
            }
            slice_begin.push_back(b);
            slice_end.push_back(b + ns);
            ++my;
            launches.fetch_add(1);
            if (my >= 2) {  // two slices in flight; inspect the older one
                const int q = (my - 2) & 1;
                if (cudaEventSynchronize(c->ev_slice[q]) != cudaSuccess) { fail(cuda_fail(cudaGetLastError(), "sync")); return; }
                harvest(q, slice_begin[my - 2], slice_end[my - 2]);
            }
        }
        if (cudaEventRecord(c->ev_stop, c->stream) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) {
            fail(cuda_fail(cudaGetLastError(), "cudaStreamSynchronize")); return;
        }
        if (my > 0) harvest((my - 1) & 1, slice_begin[my - 1], slice_end[my - 1]);
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev_start, c->ev_stop);
        dev_ms[d] = ms;
    };
    if (n == 1) {
        worker(0);
    } else {
        std::vector<std::thread> th;
        for (int d = 1; d < n; ++d) th.emplace_back(worker, d);
        worker(0);
        for (auto &t : th) t.join();
    }
    if (err.load() != ES_OK) { set_error(err_msg); return err.load(); }
    if (shared && n > 1) {  // final value of the shared word (every device has synchronised;
                            // one device's last slice already copied it back)
        CK(cudaSetDevice(cs[0]->dev));
        CK(cudaMemcpy(cs[0]->h_pin, cs[0]->d_best, 8, cudaMemcpyDeviceToHost));
        lower(cs[0]->h_pin[0]);
    }
    res->best = best.load();
    res->prefix = prefix();
    res->swept = swept.load();
    res->reason = stop_reason.load();
    res->stopped = res->reason != 0;
    res->launches = launches.load();
    res->device_ms = *std::max_element(dev_ms.begin(), dev_ms.end());
    return ES_OK;
}

// The result of a finished or stopped K1 sweep over [0, n_chunks) of `pl`.
static void k1_result(const K1Plan &pl, const SweepOut &sw, int P, es_result *r) {
    const uint64_t sentinel = 1ull << P;
    r->device_ms += sw.device_ms;
    r->launches += sw.launches;
    const uint64_t swept_patterns = std::min<uint64_t>(sw.swept * pl.patterns_per_chunk(), sentinel);
    r->patterns_swept += swept_patterns;
    r->patterns_swept = std::min(r->patterns_swept, sentinel);
    if (sw.best < sentinel) {
        r->verdict = ES_COUNTEREXAMPLE;
        r->witness_index = sw.best;
        // the minimum, unless a stop left chunks below it unswept (cofactor
        // bits above the chunk interleave high patterns into low chunks)
        const bool minimal = sw.prefix >= pl.n_chunks || sw.best < pl.first_pattern(sw.prefix);
        r->witness_minimal = minimal ? 1 : 0;
        r->patterns_evaluated = minimal ? ref_patterns_for_hit(sw.best, P) : r->patterns_swept;
    } else if (sw.stopped) {
        r->verdict = ES_BUDGET_EXCEEDED;
        r->reason = sw.reason;
        r->patterns_evaluated = r->patterns_swept;
    } else {
        r->verdict = ES_EXHAUSTED_ZERO;
        r->patterns_evaluated = sentinel;
        r->patterns_swept = sentinel;
    }
}

// ---------------------------------------------------------------------------
// K2 driver (single program or batch)
// ---------------------------------------------------------------------------

// Device record of a gate / output (16 bytes): byte offsets of the operand /
// destination slots for the launch's stride, then the K2_* flags.
static uint4 k2_record(const K2Gate &g, uint32_t stride) {
    // the complement flags are mirrored into bits 31 / 30 so the kernel turns
    // them into masks with one arithmetic shift each (copy numbers < 2^14):
    // config 4 17.8 -> 15.8 ms
    const uint32_t ctl = g.ctl | ((g.ctl & K2_NEG_A) ? 0x80000000u : 0u) | ((g.ctl & K2_NEG_B) ? 0x40000000u : 0u);
    return make_uint4(g.a * stride, g.b * stride, g.d * stride, ctl);
}

template <int W>
static int launch_k2(int grid, size_t smem, cudaStream_t st, const K2Job *jobs, const K2Item *items,
                     uint64_t begin, uint64_t end, unsigned *counter, int smem_bytes, int lanes) {
    if (lanes == 4) es_k2d<W, 4><<<grid, 128, smem, st>>>(jobs, items, begin, end, counter, smem_bytes);
    else if (lanes == 2) es_k2d<W, 2><<<grid, 128, smem, st>>>(jobs, items, begin, end, counter, smem_bytes);
    else es_k2<W><<<grid, 128, smem, st>>>(jobs, items, begin, end, counter, smem_bytes);
    CK(cudaGetLastError());
    return ES_OK;
}

template <class K>
static int k2_occ(K kern, size_t smem, int *nb) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb, kern, 128, smem));
    return ES_OK;
}

template <int W>
static int k2_occupancy(size_t smem, int *nb, int lanes) {
    if (lanes == 4) return k2_occ(es_k2d<W, 4>, smem, nb);
    if (lanes == 2) return k2_occ(es_k2d<W, 2>, smem, nb);
    return k2_occ(es_k2<W>, smem, nb);
}

// One launch group: jobs sharing a words-per-thread width W.  Items are dealt
// round-robin across jobs (item r of every job before item r+1 of any job),
// so a non-equivalent job's first item settles its minimum before its later
// items are claimed -- those are then skipped -- while every item below the
// final minimum is still fully evaluated.
struct K2Group {
    std::vector<int> jobs_idx;   // indices into the caller's job arrays
    int W = 1, smem_bytes = 0, nb = 1;
    int lanes = 1;               // multi-lane programs (es_k2d) when > 1
    size_t smem = 0;
    uint4 *code = nullptr;       // device-image records, in the pinned stage
    size_t n_code = 0;
    std::vector<K2Job> jobs;
    std::vector<K2Item> items;
    std::vector<unsigned long long> h_best;
    std::vector<unsigned> h_swept;   // per job: items evaluated
    std::vector<uint64_t> n_items, item_words;
    uint8_t *d_buf = nullptr;
    K2Job *d_jobs = nullptr;
    K2Item *d_items = nullptr;
    unsigned long long *d_best = nullptr;
    unsigned *d_swept = nullptr;
    uint64_t done_items = 0;
    int launches = 0;
};

static int k2_target_ctas() {
    const char *e = getenv("ES_K2_CTAS");
    return e ? std::max(1, atoi(e)) : 2;
}

static int k2_group_prepare(K2Group &gp, const es_prog *progs, const K2Prog *const *kps, Ctx *c,
                            uint4 *stage, cudaStream_t st) {
    const int T = 128;
    const std::vector<int> &group = gp.jobs_idx;
    int max_slots = 1;
    for (int j : group) max_slots = std::max(max_slots, kps[j]->num_slots);
    int dev_smem = 0;
    CK(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev));
    auto smem_for = [&](int W) {  // the largest job's slot file + records (kernel layout)
        size_t m = 16;
        for (int j : group)
            m = std::max(m, (size_t)std::max(kps[j]->num_slots, 1) * T * W * 4 + (k2_device_records(*kps[j]) + kK2PadRecords) * 16);
        return m;
    };
    // widest W that keeps the target number of resident CTAs per SM, else
    // fewer CTAs (the interpreter is latency-bound: warps matter more than W)
    int W = 0;
    for (int ctas = k2_target_ctas(); ctas >= 1 && !W; --ctas)
        for (int cand : {4, 2, 1})
            if ((size_t)ctas * (smem_for(cand) + 1024) <= (size_t)dev_smem + 1024) { W = cand; break; }
    if (!W) {
        set_error("program needs " + std::to_string(max_slots) + " slots: too many for the K2 interpreter");
        return ES_E_BAD_PROGRAM;
    }
    gp.W = W;
    gp.smem = smem_for(W);
    gp.smem_bytes = (int)gp.smem;
    const uint32_t stride = (uint32_t)T * W * 4;
    const int G = (int)group.size();
    std::vector<size_t> off(G + 1, 0);  // one record per gate / output
    for (int q = 0; q < G; ++q) off[q + 1] = off[q] + k2_device_records(*kps[group[q]]);
    gp.code = stage;  // records built straight into pinned memory: one DMA, no bounce copy
    gp.n_code = off[G];
    parallel_for(G, [&](int q) {
        uint4 *dst = gp.code + off[q];
        const K2Prog &kp = *kps[group[q]];
        for (const K2Gate &g : kp.gates) {
            uint4 r = k2_record(g, stride);
            // two-lane gate records: the byte-msb masks es_k2d<W, 2> PRMTs out
            // -- NEG_A in bit 31 (k2_record), NEG_B in bit 23, XOR in bit 15
            // (for XOR the combined inversion is NEG_A and mb = 0)
            if (kp.lanes >= 2 && !(g.ctl & K2_OUT))
                r.w = (r.w & ~0x00808000u) | ((g.ctl & K2_XOR) ? 0x8000u : ((g.ctl & K2_NEG_B) ? 0x800000u : 0u));
            *dst++ = r;
        }
    });
    auto kwords = [&](int q) {  // kernel words of job q (cofactor PIs excluded)
        const int j = group[q];
        return 1ull << std::max(progs[j].num_pis - 5 - (int)kps[j]->cof_pis.size(), 0);
    };
    // the group's lane count is its programs' (build_k2prog: ES_K2_LANES)
    gp.lanes = group.empty() ? 1 : kps[group[0]]->lanes;
    for (int j : group)
        if (kps[j]->lanes != gp.lanes) { set_error("internal: K2 programs of different lane counts in one group"); return ES_E_BAD_PROGRAM; }
    int rc = W == 4 ? k2_occupancy<4>(gp.smem, &gp.nb, gp.lanes) : W == 2 ? k2_occupancy<2>(gp.smem, &gp.nb, gp.lanes)
                                                                : k2_occupancy<1>(gp.smem, &gp.nb, gp.lanes);
    if (rc != ES_OK) return rc;
    gp.nb = std::max(gp.nb, 1);
    // item size: 4096 words, halved (down to one CTA iteration) until the
    // group has >= 8 items per resident CTA
    uint64_t iw = 4096;
    for (;;) {
        uint64_t cnt = 0;
        for (int q = 0; q < G; ++q) {
            const uint64_t tw = kwords(q);
            cnt += (tw + std::min(tw, iw) - 1) / std::min(tw, iw);
        }
        if (cnt >= (uint64_t)c->sms * gp.nb * 8 || iw <= (uint64_t)T * W) break;
        iw >>= 1;
    }
    gp.jobs.assign(G, K2Job{});
    gp.h_best.assign(G, 0);
    gp.n_items.assign(G, 0);
    gp.item_words.assign(G, 0);
    uint64_t max_items = 0;
    for (int q = 0; q < G; ++q) {
        const int P = progs[group[q]].num_pis;
        const uint64_t tw = kwords(q);
        gp.item_words[q] = std::min<uint64_t>(tw, iw);
        gp.n_items[q] = (tw + gp.item_words[q] - 1) / gp.item_words[q];
        max_items = std::max(max_items, gp.n_items[q]);
        gp.h_best[q] = 1ull << P;
    }
    gp.items.clear();
    for (uint64_t r = 0; r < max_items; ++r)
        for (int q = 0; q < G; ++q)
            if (r < gp.n_items[q]) {
                const uint64_t tw = kwords(q);
                const uint64_t w0 = r * gp.item_words[q];
                gp.items.push_back(K2Item{w0, (unsigned)std::min<uint64_t>(gp.item_words[q], tw - w0), q});
            }
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t code_b = std::max<size_t>(gp.n_code, 1) * sizeof(uint4);
    const size_t jobs_b = (size_t)G * sizeof(K2Job);
    const size_t items_b = std::max<size_t>(gp.items.size(), 1) * sizeof(K2Item);
    const size_t best_b = (size_t)G * 8, swept_b = (size_t)G * 4;
    CK(cudaMallocAsync(&gp.d_buf, al(code_b) + al(jobs_b) + al(items_b) + al(best_b) + al(swept_b), st));
    uint4 *d_code = (uint4 *)gp.d_buf;
    gp.d_jobs = (K2Job *)(gp.d_buf + al(code_b));
    gp.d_items = (K2Item *)(gp.d_buf + al(code_b) + al(jobs_b));
    gp.d_best = (unsigned long long *)(gp.d_buf + al(code_b) + al(jobs_b) + al(items_b));
    gp.d_swept = (unsigned *)(gp.d_buf + al(code_b) + al(jobs_b) + al(items_b) + al(best_b));
    gp.h_swept.assign(G, 0u);
    for (int q = 0; q < G; ++q) {
        const int j = group[q];
        K2Job &J = gp.jobs[q];
        J.code = d_code + off[q];
        J.best = gp.d_best + q;
        J.swept = gp.d_swept + q;
        J.total_words = kwords(q);
        J.n_recs = (int)k2_device_records(*kps[j]);
        J.num_pis = progs[j].num_pis;
        J.valid_mask = lane_valid_mask(progs[j].num_pis);
        J.cof_n = (int)kps[j]->cof_pis.size();
        J.cof_mask = 0;
        for (int b = 0; b < J.cof_n; ++b) {
            J.cof_pos[b] = (unsigned char)(kps[j]->cof_pis[b] - 1);
            J.cof_mask |= 1ull << kps[j]->cof_pis[b];
        }
    }
    return ES_OK;
}

// the group's image to the device (after k2_group_prepare, same stream)
static int k2_group_upload(K2Group &gp, cudaStream_t st) {
    CK(cudaMemcpyAsync((uint4 *)gp.d_buf, gp.code, gp.n_code * sizeof(uint4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(gp.d_jobs, gp.jobs.data(), gp.jobs.size() * sizeof(K2Job), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(gp.d_items, gp.items.data(), gp.items.size() * sizeof(K2Item), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(gp.d_best, gp.h_best.data(), gp.h_best.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(gp.d_swept, 0, gp.h_swept.size() * 4, st));
    return ES_OK;
}

static int k2_group_launch(K2Group &gp, cudaStream_t st, unsigned *counter, uint64_t begin,
                           uint64_t end, int sms) {
    CK(cudaMemsetAsync(counter, 0, sizeof(unsigned), st));
    const int grid = (int)std::min<uint64_t>(end - begin, (uint64_t)sms * gp.nb);
    const int rc = gp.W == 4 ? launch_k2<4>(grid, gp.smem, st, gp.d_jobs, gp.d_items, begin, end, counter, gp.smem_bytes, gp.lanes)
                 : gp.W == 2 ? launch_k2<2>(grid, gp.smem, st, gp.d_jobs, gp.d_items, begin, end, counter, gp.smem_bytes, gp.lanes)
                             : launch_k2<1>(grid, gp.smem, st, gp.d_jobs, gp.d_items, begin, end, counter, gp.smem_bytes, gp.lanes);
    if (rc == ES_OK) { gp.launches++; gp.done_items = end; }
    return rc;
}

// first pattern (copy 0) of kernel word w of a job: k2_expand on the host
static uint64_t k2_expand_host(uint64_t w, const K2Job &job) {
    uint64_t x = w << 5;
    for (int i = 0; i < job.cof_n; ++i) {
        const unsigned s = job.cof_pos[i];
        x = ((x >> s) << (s + 1)) | (x & ((1ull << s) - 1ull));
    }
    return x;
}

static void k2_group_results(const K2Group &gp, const es_prog *progs, const K2Prog *const *kps,
                             bool stopped, int stop_reason, es_result *outs) {
    const int G = (int)gp.jobs_idx.size();
    std::vector<uint64_t> done_cnt(G, 0);
    if (gp.done_items >= gp.items.size()) done_cnt = gp.n_items;
    else
        for (uint64_t x = 0; x < gp.done_items; ++x) done_cnt[gp.items[x].job]++;
    for (int q = 0; q < G; ++q) {
        const int j = gp.jobs_idx[q];
        es_result *r = &outs[j];
        const int P = progs[j].num_pis;
        const uint64_t sentinel = 1ull << P;
        r->engine = ES_ENGINE_INTERP;
        r->launches += gp.launches;
        r->num_luts = (int)kps[j]->gates.size();
        r->regs_per_thread = gp.W;  // K2: words per thread
        const uint64_t covered = done_cnt[q];  // this job's items in completed launches
        const uint64_t item_patterns = (gp.item_words[q] * 32) << kps[j]->cof_pis.size();
        // items evaluated (skipped ones excluded), the last possibly partial
        const uint64_t swept = std::min<uint64_t>((uint64_t)gp.h_swept[q] * item_patterns, sentinel);
        if (gp.h_best[q] < sentinel) {
            r->verdict = ES_COUNTEREXAMPLE;
            r->witness_index = gp.h_best[q];
            r->patterns_swept = swept;
            // a job's completed items are a prefix of its items (round-robin
            // order); the witness is the minimum unless a stop left an item
            // whose first pattern lies below it (cofactor bits above the item)
            const bool minimal = covered >= gp.n_items[q] ||
                                 gp.h_best[q] < k2_expand_host(covered * gp.item_words[q], gp.jobs[q]);
            r->witness_minimal = minimal ? 1 : 0;
            r->patterns_evaluated = minimal ? ref_patterns_for_hit(gp.h_best[q], P) : r->patterns_swept;
        } else if (stopped && covered < gp.n_items[q]) {
            r->verdict = ES_BUDGET_EXCEEDED;
            r->reason = stop_reason;
            r->patterns_evaluated = std::min<uint64_t>(covered * item_patterns, sentinel);
            r->patterns_swept = swept;
        } else {
            r->verdict = ES_EXHAUSTED_ZERO;
            r->patterns_evaluated = sentinel;
            r->patterns_swept = swept;
        }
    }
}

// ---------------------------------------------------------------- K4
// Which interpreter jobs get a straight-line body: num_pis >= ES_K4_MIN_PIS
// (default 18; ES_K4=0 turns K4 off).  Smaller jobs' sweeps are a few items
// and the body's host cost (mapping + lowering, ~1 ms of one core) would not
// pay.  Measured on config 4 (device ms, best of 4): min 16 / 18 / 20 / 22 ->
// 1.88 / 1.91 / 2.39 / 3.56 (240K-slot modules; K2 alone 11.6).
static int k4_min_pis() {
    static const int v = [] {
        const char *e = getenv("ES_K4");
        if (e && atoi(e) == 0) return 1 << 20;
        const char *m = getenv("ES_K4_MIN_PIS");
        return m ? atoi(m) : 18;
    }();
    return v;
}

// A loaded module and, per device, its job table + items (position-
// independent, uploaded once) and the per-job sentinels best starts from
struct K4Img {
    int dev = -1;
    uint8_t *d_img = nullptr;                  // jobs, then items
    unsigned long long *d_best0 = nullptr;     // per job: 2^num_pis
};
struct K4Mod {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    int variant = 0, blocks = 1;
    int G = 0;
    std::vector<uint64_t> n_items;
    std::vector<K4JobD> jobs;
    std::vector<K2Item> items;
    std::vector<K4Img> imgs;
    int users = 0;  // runs holding it (under g_k4_mu)
};
static std::mutex g_k4_mu;
static double g_k4_t[3];  // ES_VERBOSE: ms in module build / library load / context load
static std::unordered_map<uint64_t, std::unique_ptr<K4Mod>> g_k4_mods;  // key: the bodies' hashes
// bound on loaded modules (~2.3 MB of code each): a long sweep makes new
// ones every round; modules no run holds are unloaded past it
constexpr size_t kK4MaxModules = 192;

static void k4_evict_locked() {
    if (g_k4_mods.size() <= kK4MaxModules) return;
    for (auto it = g_k4_mods.begin(); it != g_k4_mods.end() && g_k4_mods.size() > kK4MaxModules / 2;) {
        K4Mod &m = *it->second;
        if (m.users) { ++it; continue; }
        for (K4Img &x : m.imgs) cudaFree(x.d_img);
        cudaLibraryUnload(m.lib);
        it = g_k4_mods.erase(it);
    }
}

// a run's hold on its modules (released when the run ends)
struct K4Hold {
    std::vector<K4Mod *> mods;
    ~K4Hold() {
        std::lock_guard<std::mutex> lk(g_k4_mu);
        for (K4Mod *m : mods) --m->users;
    }
};

// one module launch of a run: its cached module and this run's scratch
struct K4Launch {
    std::vector<int> jobs_idx;
    K4Mod *mod = nullptr;
    const K4Img *img = nullptr;
    size_t scratch_job0 = 0;  // first job slot of the run's best / swept arrays
    int instrs = 0;
};

static uint64_t hash_words(const std::vector<uint64_t> &w) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ w.size();
    for (uint64_t x : w) {
        h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xff51afd7ed558ccdull;
    }
    return h;
}

// a module's host image: job table and items of kK4ItemWords words (a CTA
// claims one and runs kK4ItemWords / 256 body calls per thread; fixed 4096
// measured 2.48 ms on config 4 against 1.76 with K2's halving rule, 8192 /
// 16384: 3.27 / 3.78).  Order:
// every job's first item round-robin -- a non-equivalent job usually settles
// its minimum there and its later items are skipped -- then the rest job by
// job, so the CTAs sweeping a job share its body in L2 (job-major
// throughout measured 1.9x slower on config 4: non-equivalent jobs' items
// claimed before their minimum lands)
constexpr uint64_t kK4ItemWords = 4096;
static void k4_image(K4Mod &m, const std::vector<int> &jobs_idx, const es_prog *progs,
                     const K2Prog *const *kps, int sms) {
    const int G = (int)jobs_idx.size();
    m.G = G;
    auto kwords = [&](int q) {
        const int j = jobs_idx[q];
        return 1ull << std::max(progs[j].num_pis - 5 - (int)kps[j]->cof_pis.size(), 0);
    };
    // halved (down to one CTA pass) until the module has >= 8 items per resident CTA
    uint64_t iw = getenv("ES_K4_ITEM") ? (uint64_t)atoi(getenv("ES_K4_ITEM")) : kK4ItemWords;
    for (;;) {
        uint64_t cnt = 0;
        for (int q = 0; q < G; ++q) {
            const uint64_t tw = kwords(q);
            cnt += (tw + std::min(tw, iw) - 1) / std::min(tw, iw);
        }
        if (cnt >= (uint64_t)sms * 8 || iw <= 256) break;
        iw >>= 1;
    }
    m.jobs.assign(G, K4JobD{});
    m.n_items.assign(G, 0);
    for (int q = 0; q < G; ++q) {
        const int j = jobs_idx[q];
        K4JobD &J = m.jobs[q];
        J.total_words = kwords(q);
        J.valid_mask = lane_valid_mask(progs[j].num_pis);
        J.body = (unsigned)q;
        J.cof_n = (int)kps[j]->cof_pis.size();
        for (int b = 0; b < J.cof_n; ++b) J.cof_pos[b] = (unsigned char)(kps[j]->cof_pis[b] - 1);
    }
    m.items.clear();
    for (int q = 0; q < G; ++q) {
        const uint64_t tw = kwords(q);
        m.items.push_back(K2Item{0, (unsigned)std::min(tw, iw), q});
        m.n_items[q] = 1;
    }
    for (int q = 0; q < G; ++q) {
        const uint64_t tw = kwords(q);
        for (uint64_t w0 = std::min(tw, iw); w0 < tw; w0 += iw) {
            m.items.push_back(K2Item{w0, (unsigned)std::min(iw, tw - w0), q});
            m.n_items[q]++;
        }
    }
}

// K4 bodies of the jobs that lack one, on all host cores (a job whose body
// does not fit gets ok = false and stays on K2)
static void k4_build_bodies(const es_prog *progs, const K2Prog *const *kps, const std::vector<int> &jobs) {
    std::vector<int> todo;
    for (int j : jobs)
        if (!kps[j]->k4) todo.push_back(j);
    parallel_for((int)todo.size(), [&](int q) {
        const int j = todo[q];
        const K2Prog &kp = *kps[j];
        auto b = std::make_shared<K4Body>();
        Dag dag;
        std::string err;
        if (build_dag(progs[j], &dag, &err) == ES_OK) {
            LutNet net;
            map_cofactored(dag, kp.cof_pis, &net);
            SassStats st;
            if (k4_body(net, -1, &b->code, &st, &b->variant, &err)) {
                b->ok = true;
                b->instrs = st.instrs;
                b->hash = hash_words(b->code);
            }
        }
        kp.k4 = b;
    }, 1);
}

// es_batch_prepare: the bodies of the jobs K4 would take, ahead of the first run
void k4_prebuild(int n, const es_prog *progs, const K2Prog *const *kps) {
    std::vector<int> cand;
    for (int j = 0; j < n; ++j)
        if (kps[j] && progs[j].num_pis >= k4_min_pis() && k2_fits(*kps[j])) cand.push_back(j);
    k4_build_bodies(progs, kps, cand);
}

// bodies for the candidate jobs (built once per program, in parallel), then
// modules of up to k4_max_bodies() bodies; each module is built, loaded and
// imaged on the device once (cached by its bodies' hashes), so a warm run
// only looks them up
static int k4_prepare(const es_prog *progs, const K2Prog *const *kps, const std::vector<int> &cand, Ctx *c,
                      std::vector<K4Launch> *mods, K4Hold *hold) {
    NvtxRange nvtx("es_k4_prepare");
    k4_build_bodies(progs, kps, cand);
    int variant = 0;
    K4Launch cur;
    int slots = 0;
    size_t job0 = 0;
    std::vector<const std::vector<uint64_t> *> bodies;
    auto flush = [&]() -> int {
        if (cur.jobs_idx.empty()) return ES_OK;
        // (the body fixes the logic; the word count and copy layout come
        // from num_pis and the cofactor PIs, which an unused PI leaves out
        // of the code)
        uint64_t key = 0x84222325CBF29CE4ull;
        for (int j : cur.jobs_idx) {
            key = (key ^ kps[j]->k4->hash) * 0x100000001B3ull + 0x9E37;
            key = (key ^ (uint64_t)progs[j].num_pis) * 0x100000001B3ull;
            for (int32_t pi : kps[j]->cof_pis) key = (key ^ (uint64_t)pi) * 0x100000001B3ull;
        }
        std::lock_guard<std::mutex> lk(g_k4_mu);
        auto it = g_k4_mods.find(key);
        if (it == g_k4_mods.end()) {
            k4_evict_locked();
            std::vector<char> cubin;
            std::vector<uint32_t> entry;
            std::string err;
            const double ta = now_ms();
            if (!k4_module(bodies, variant, &cubin, &entry, &err)) { set_error(err); return ES_E_CUDA; }
            auto m = std::make_unique<K4Mod>();
            const double tb = now_ms();
            CK(cudaLibraryLoadData(&m->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
            CK(cudaLibraryGetKernel(&m->kern, m->lib, "es_k4"));
            g_k4_t[0] += tb - ta;
            g_k4_t[1] += now_ms() - tb;
            m->variant = variant;
            m->blocks = k4_blocks(variant);
            k4_image(*m, cur.jobs_idx, progs, kps, c->sms * m->blocks);
            it = g_k4_mods.emplace(key, std::move(m)).first;
        }
        K4Mod &m = *it->second;
        const K4Img *img = nullptr;
        for (const K4Img &x : m.imgs)
            if (x.dev == c->dev) img = &x;
        if (!img) {
            // load the module into this context now (lazy loading would do it
            // inside the first launch) and upload its image
            cudaFuncAttributes fa;
            const double tc = now_ms();
            CK(cudaFuncGetAttributes(&fa, (const void *)m.kern));
            g_k4_t[2] += now_ms() - tc;
            K4Img x;
            x.dev = c->dev;
            const size_t jb = ((size_t)m.G * sizeof(K4JobD) + 255) & ~(size_t)255;
            const size_t ib = m.items.size() * sizeof(K2Item);
            CK(cudaMalloc(&x.d_img, jb + ib + (size_t)m.G * 8));
            CK(cudaMemcpy(x.d_img, m.jobs.data(), (size_t)m.G * sizeof(K4JobD), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(x.d_img + jb, m.items.data(), ib, cudaMemcpyHostToDevice));
            x.d_best0 = (unsigned long long *)(x.d_img + jb + ib);
            std::vector<unsigned long long> b0(m.G);
            for (int q = 0; q < m.G; ++q) b0[q] = 1ull << progs[cur.jobs_idx[q]].num_pis;
            CK(cudaMemcpy(x.d_best0, b0.data(), b0.size() * 8, cudaMemcpyHostToDevice));
            m.imgs.push_back(x);
            img = &m.imgs.back();
        }
        ++m.users;
        hold->mods.push_back(&m);
        cur.mod = &m;
        cur.img = img;
        cur.scratch_job0 = job0;
        job0 += cur.jobs_idx.size();
        mods->push_back(std::move(cur));
        cur = K4Launch();
        bodies.clear();
        slots = 0;
        return ES_OK;
    };
    for (variant = 0; variant < k4_variants(); ++variant) {  // one run of modules per template variant
        const int cap = k4_body_capacity(variant), maxb = k4_max_bodies(variant);
        for (int j : cand) {
            const K4Body &b = *kps[j]->k4;
            if (!b.ok || b.variant != variant) continue;
            const int need = (int)b.code.size() / 2 + 1;
            if (!cur.jobs_idx.empty() && ((int)cur.jobs_idx.size() >= maxb || slots + need > cap)) {
                int rc = flush();
                if (rc != ES_OK) return rc;
            }
            cur.jobs_idx.push_back(j);
            bodies.push_back(&b.code);
            slots += need;
            cur.instrs += b.instrs;
        }
        int rc = flush();
        if (rc != ES_OK) return rc;
    }
    return ES_OK;
}

// the run's scratch for every module (best from the modules' sentinels,
// swept and counters zero), then one launch per module, all on `st`
struct K4Scratch {
    uint8_t *d = nullptr;
    unsigned long long *best = nullptr;
    unsigned *swept = nullptr, *counter = nullptr;
    std::vector<unsigned long long> h_best;
    std::vector<unsigned> h_swept;
};
constexpr int kK4Streams = 4;  // module launches round-robin over side[3..6]: one module's tail overlaps the next
static int k4_launch_all(std::vector<K4Launch> &mods, K4Scratch &sc, Ctx *c, cudaStream_t st) {
    size_t nj = 0;
    for (const K4Launch &m : mods) nj += m.jobs_idx.size();
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    CK(cudaMallocAsync(&sc.d, al(nj * 8) + al(nj * 4) + al(mods.size() * 4), st));
    sc.best = (unsigned long long *)sc.d;
    sc.swept = (unsigned *)(sc.d + al(nj * 8));
    sc.counter = (unsigned *)(sc.d + al(nj * 8) + al(nj * 4));
    CK(cudaMemsetAsync(sc.swept, 0, al(nj * 4) + al(mods.size() * 4), st));
    for (const K4Launch &m : mods)
        CK(cudaMemcpyAsync(sc.best + m.scratch_job0, m.img->d_best0, m.jobs_idx.size() * 8,
                           cudaMemcpyDeviceToDevice, st));
    CK(cudaEventRecord(c->ev_side[3], st));
    for (int q = 1; q < kK4Streams; ++q) CK(cudaStreamWaitEvent(c->side[3 + q], c->ev_side[3], 0));
    for (size_t i = 0; i < mods.size(); ++i) {
        const K4Launch &m = mods[i];
        const size_t jb = ((size_t)m.mod->G * sizeof(K4JobD) + 255) & ~(size_t)255;
        K4ParamsD p{(const K4JobD *)m.img->d_img, (const K2Item *)(m.img->d_img + jb),
                    (unsigned long long)m.mod->items.size(), sc.best + m.scratch_job0, sc.swept + m.scratch_job0,
                    sc.counter + i, 1u};
        void *args[] = {&p};
        const int grid = (int)std::min<uint64_t>(m.mod->items.size(), (uint64_t)c->sms * m.mod->blocks);
        CK(cudaLaunchKernel((const void *)m.mod->kern, dim3(grid), dim3(256), args, 0,
                            c->side[3 + (int)(i % kK4Streams)]));
    }
    for (int q = 0; q < kK4Streams; ++q) CK(cudaEventRecord(c->ev_side[3 + q], c->side[3 + q]));
    sc.h_best.resize(nj);
    sc.h_swept.resize(nj);
    return ES_OK;
}

// es_result of the modules' jobs (a whole, unsliced launch: k2_group_results'
// rules with every item completed)
static void k4_results(const std::vector<K4Launch> &mods, const K4Scratch &sc, const es_prog *progs,
                       const K2Prog *const *kps, es_result *outs) {
    for (const K4Launch &m : mods)
        for (size_t q = 0; q < m.jobs_idx.size(); ++q) {
            const int j = m.jobs_idx[q];
            es_result *r = &outs[j];
            const int P = progs[j].num_pis;
            const uint64_t sentinel = 1ull << P;
            const unsigned long long best = sc.h_best[m.scratch_job0 + q];
            r->engine = ES_ENGINE_JIT;
            r->launches += 1;
            r->num_luts = kps[j]->k4->instrs;
            r->regs_per_thread = 255;
            // swept = kernel words of the evaluated items, each 32 patterns x 2^k copies
            r->patterns_swept = std::min<uint64_t>(((uint64_t)sc.h_swept[m.scratch_job0 + q] * 32)
                                                       << kps[j]->cof_pis.size(), sentinel);
            if (best < sentinel) {
                r->verdict = ES_COUNTEREXAMPLE;
                r->witness_index = best;
                r->witness_minimal = 1;
                r->patterns_evaluated = ref_patterns_for_hit(best, P);
            } else {
                r->verdict = ES_EXHAUSTED_ZERO;
                r->patterns_evaluated = sentinel;
            }
        }
}

static int run_k2(int n_jobs, const es_prog *progs, const std::vector<int> &active_in,
                  const es_run_opts &o, Ctx *c, double deadline, es_result *outs,
                  const K2Prog *const *prebuilt = nullptr, std::vector<int> *unfit = nullptr) {
    NvtxRange nvtx("es_k2");
    // host: K2 programs (schedule, accumulator forwarding), in parallel --
    // unless the caller built them already (sub-miter batches do at extraction)
    std::vector<K2Prog> own;
    std::vector<int> bad(n_jobs, 0);
    if (!prebuilt) {
        own.resize(n_jobs);
        std::vector<K2Prog> &kps = own;
        std::atomic<size_t> next{0};
        auto work = [&]() {
            for (;;) {
                const size_t q = next.fetch_add(1);
                if (q >= active_in.size()) return;
                const int j = active_in[q];
                Dag dag;
                std::string err;
                if (build_dag(progs[j], &dag, &err) != ES_OK) { bad[j] = 1; continue; }
                build_k2prog_auto(dag, &kps[j]);
            }
        };
        const int nt = (int)std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()),
                                             std::max<size_t>(1, active_in.size() / 64));
        std::vector<std::thread> th;
        for (int q = 1; q < nt; ++q) th.emplace_back(work);
        work();
        for (auto &x : th) x.join();
    }
    for (int j : active_in)
        if (bad[j]) { set_error("malformed program in batch (job " + std::to_string(j) + ")"); return ES_E_BAD_PROGRAM; }
    std::vector<const K2Prog *> own_ptr;
    if (!prebuilt) {
        own_ptr.resize(n_jobs, nullptr);
        for (int j : active_in) own_ptr[j] = &own[j];
    }
    const K2Prog *const *kps = prebuilt ? prebuilt : own_ptr.data();
    // programs whose slot file cannot fit one CTA's shared memory: handed back
    // to the caller for K1 (or an error when the caller forced the interpreter)
    std::vector<int> active;
    active.reserve(active_in.size());
    for (int j : active_in) {
        if (k2_fits(*kps[j])) { active.push_back(j); continue; }
        if (!unfit) {
            set_error("program needs " + std::to_string(kps[j]->num_slots) +
                      " slots: too many for the K2 interpreter (job " + std::to_string(j) + ")");
            return ES_E_BAD_PROGRAM;
        }
        unfit->push_back(j);
    }
    if (active.empty()) return ES_OK;
    const bool sliced = deadline >= 0 || o.cancel_flag != nullptr;
    // K4: jobs with enough words get a straight-line body (one launch per
    // module of bodies, on its own stream, concurrent with the K2 groups)
    std::vector<K4Launch> k4mods;
    K4Hold k4hold;
    K4Scratch k4sc;
    double t_k4 = 0;
    if (!sliced && o.engine != ES_ENGINE_INTERP) {
        std::vector<int> cand;
        for (int j : active)
            if (progs[j].num_pis >= k4_min_pis()) cand.push_back(j);
        if (!cand.empty()) {
            const double tk = now_ms();
            int rc = k4_prepare(progs, kps, cand, c, &k4mods, &k4hold);
            if (rc != ES_OK) return rc;
            std::vector<uint8_t> on_k4(n_jobs, 0);
            for (const K4Launch &m : k4mods)
                for (int j : m.jobs_idx) on_k4[j] = 1;
            active.erase(std::remove_if(active.begin(), active.end(), [&](int j) { return on_k4[j] != 0; }),
                         active.end());
            t_k4 = now_ms() - tk;
        }
    }
    if (active.empty() && k4mods.empty()) return ES_OK;
    // launch groups by slot count: small programs get 4 words per thread
    std::vector<K2Group> groups(3);
    for (int j : active) {
        const int sl = kps[j]->num_slots;
        groups[k2_group_of(sl, k2_device_records(*kps[j]))].jobs_idx.push_back(j);
    }
    groups.erase(std::remove_if(groups.begin(), groups.end(),
                                [](const K2Group &g) { return g.jobs_idx.empty(); }),
                 groups.end());
    const bool verbose = getenv("ES_VERBOSE") != nullptr;
    const double t0 = now_ms();
    size_t total_recs = 0;
    for (const K2Group &gp : groups)
        for (int j : gp.jobs_idx) total_recs += k2_device_records(*kps[j]);
    if (total_recs > c->stage_cap) {
        if (c->h_stage) CK(cudaFreeHost(c->h_stage));
        c->h_stage = nullptr;
        const size_t cap = std::max(total_recs, c->stage_cap + c->stage_cap / 2);
        CK(cudaMallocHost(&c->h_stage, cap * sizeof(uint4)));
        c->stage_cap = cap;
    }
    bool stopped = false;
    int stop_reason = 0;
    float dev_ms = 0;
    std::vector<size_t> stage_off(groups.size() + 1, 0);
    for (size_t g = 0; g < groups.size(); ++g) {  // records of each group straight into pinned memory
        size_t n = 0;
        for (int j : groups[g].jobs_idx) n += k2_device_records(*kps[j]);
        stage_off[g + 1] = stage_off[g] + n;
    }
    double t1 = now_ms();
    if (sliced) {  // host images + one upload phase, then slices
        for (size_t g = 0; g < groups.size(); ++g) {
            int rc = k2_group_prepare(groups[g], progs, kps, c, c->h_stage + stage_off[g], c->stream);
            if (rc == ES_OK) rc = k2_group_upload(groups[g], c->stream);
            if (rc != ES_OK) return rc;
        }
        t1 = now_ms();
        CK(cudaEventRecord(c->ev_start, c->stream));
    }
    if (!sliced) {
        // all groups at once, one side stream each, each launched as soon as
        // its host image is ready, the largest programs first (their group is
        // the long pole; the smaller groups' host work overlaps it); device
        // time = makespan from the first upload.  K4 modules go first, in
        // turn on their own stream.
        if (!k4mods.empty()) {
            t1 = now_ms();
            CK(cudaEventRecord(c->ev_start, c->stream));
            CK(cudaStreamWaitEvent(c->side[3], c->ev_start, 0));
            int rc = k4_launch_all(k4mods, k4sc, c, c->side[3]);
            if (rc != ES_OK) return rc;
        }
        for (size_t gi = 0; gi < groups.size(); ++gi) {
            const size_t g = groups.size() - 1 - gi;
            int rc = k2_group_prepare(groups[g], progs, kps, c, c->h_stage + stage_off[g], c->stream);
            if (rc != ES_OK) return rc;
            if (gi == 0 && k4mods.empty()) {
                t1 = now_ms();
                CK(cudaEventRecord(c->ev_start, c->stream));
            }
            CK(cudaEventRecord(c->ev_side[g], c->stream));  // after the group's allocation
            CK(cudaStreamWaitEvent(c->side[g], c->ev_side[g], 0));
            rc = k2_group_upload(groups[g], c->side[g]);
            if (rc != ES_OK) return rc;
            rc = k2_group_launch(groups[g], c->side[g], c->d_counter + g, 0,
                                     groups[g].items.size(), c->sms);
            if (rc != ES_OK) return rc;
            CK(cudaEventRecord(c->ev_side[g], c->side[g]));
        }
        // join only now: a join inside the loop would order the next group's
        // allocation (on the main stream) after this group's kernel
        for (size_t g = 0; g < groups.size(); ++g) CK(cudaStreamWaitEvent(c->stream, c->ev_side[g], 0));
        if (!k4mods.empty())
            for (int q = 0; q < kK4Streams; ++q) CK(cudaStreamWaitEvent(c->stream, c->ev_side[3 + q], 0));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t g = 0; g < groups.size(); ++g) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, c->ev_start, c->ev_side[g]));
            dev_ms = std::max(dev_ms, ms);
        }
        if (!k4mods.empty())
            for (int q = 0; q < kK4Streams; ++q) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, c->ev_start, c->ev_side[3 + q]));
                dev_ms = std::max(dev_ms, ms);
            }
    } else {
        // budget / cancel: groups in turn, in slices, checking between slices
        for (K2Group &gp : groups) {
            const uint64_t NI = gp.items.size();
            const uint64_t per_slice = std::max<uint64_t>((uint64_t)c->sms * gp.nb * 8, 1);
            for (uint64_t begin = 0; begin < NI && !stopped; begin += per_slice) {
                if (stop_requested(o, deadline, &stop_reason)) { stopped = true; break; }
                int rc = k2_group_launch(gp, c->stream, c->d_counter, begin, std::min(NI, begin + per_slice), c->sms);
                if (rc != ES_OK) return rc;
                CK(cudaStreamSynchronize(c->stream));
            }
        }
        CK(cudaEventRecord(c->ev_stop, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaEventElapsedTime(&dev_ms, c->ev_start, c->ev_stop));
    }
    for (K2Group &gp : groups) {
        CK(cudaMemcpyAsync(gp.h_best.data(), gp.d_best, gp.h_best.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(gp.h_swept.data(), gp.d_swept, gp.h_swept.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaFreeAsync(gp.d_buf, c->stream));
    }
    if (!k4mods.empty()) {
        CK(cudaMemcpyAsync(k4sc.h_best.data(), k4sc.best, k4sc.h_best.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(k4sc.h_swept.data(), k4sc.swept, k4sc.h_swept.size() * 4, cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaFreeAsync(k4sc.d, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (K2Group &gp : groups) k2_group_results(gp, progs, kps, stopped, stop_reason, outs);
    if (!k4mods.empty()) k4_results(k4mods, k4sc, progs, kps, outs);
    for (int j : active) outs[j].device_ms = dev_ms;
    for (const K4Launch &m : k4mods)
        for (int j : m.jobs_idx) outs[j].device_ms = dev_ms;
    if (verbose && !k4mods.empty()) {
        float ms = -1;
        for (int q = 0; q < kK4Streams; ++q) {
            float x = -1;
            cudaEventElapsedTime(&x, c->ev_start, c->ev_side[3 + q]);
            ms = std::max(ms, x);
        }
        size_t nj = 0, ni = 0;
        int ins = 0;
        for (const K4Launch &m : k4mods) { nj += m.jobs_idx.size(); ni += m.mod->items.size(); ins += m.instrs; }
        fprintf(stderr, "[es k4] modules=%zu jobs=%zu items=%zu body-instrs=%d | bodies+modules %.2fms, "
                        "K4 %.2fms | cumulative build %.1f load %.1f ctx-load %.1f ms\n", k4mods.size(), nj, ni,
                ins, t_k4, ms, g_k4_t[0], g_k4_t[1], g_k4_t[2]);
    }
    if (verbose)
        for (size_t g = 0; g < groups.size(); ++g) {
            const K2Group &gp = groups[g];
            float gms = -1;
            if (!sliced) cudaEventElapsedTime(&gms, c->ev_start, c->ev_side[g]);
            int cof = 0;
            for (int j : gp.jobs_idx) cof += (int)kps[j]->cof_pis.size();
            fprintf(stderr, "[es k2] group W=%d jobs=%zu items=%zu records=%zu mean-k=%.2f | host+upload "
                            "%.2fms, this group %.2fms, makespan %.2fms\n", gp.W, gp.jobs_idx.size(),
                    gp.items.size(), gp.n_code, (double)cof / std::max<size_t>(1, gp.jobs_idx.size()),
                    t1 - t0, gms, dev_ms);
        }
    return ES_OK;
}

// ---------------------------------------------------------------------------
// public drivers
// ---------------------------------------------------------------------------
// Mapped programs cached by a hash of the program arrays: a warm call skips
// graph rebuild, mapping, PTX emission and the JIT-cache lookup.
struct MappedProg {
    std::vector<uint8_t> sig;        // the program arrays: a cache hit must match them exactly
    Dag dag;
    int G = 0;
    // K1 variants keyed by their cofactor PI set (ascending; empty = one word
    // per iteration), mapped on demand; kernels per (set, CTA size)
    // (cofactor PIs, copies: 0 = all 2^k, t = the restricted variant of copies 0..t-1)
    using VariantKey = std::pair<std::vector<int32_t>, int>;
    std::map<VariantKey, std::unique_ptr<LutNet>> nets;
    std::map<std::pair<VariantKey, int>, JitKernel *> jks;
    std::map<int, std::vector<int32_t>> ranks;  // max_pi -> the cheapest word PIs (<= max_pi), by fanout
    int runs = 0;                    // K1 runs so far (the reuse estimate of the auto policy)
    int batch_k = -1, batch_opt = 0; // the depth / build a batch's compile thread chose (run_batch_jit)
    std::shared_ptr<K2Prog> k2;      // interpreter program (its own cofactor depth), on demand
    bool k2_searched = false;        // built with the cofactor-depth search
    int k2_runs = 0;
    std::mutex mu;
    // the k word PIs of smallest transitive fanout among PIs <= max_pi, ascending
    std::vector<int32_t> ranked(int k, int max_pi = 1 << 20) {  // caller holds mu
        auto it = ranks.find(max_pi);
        if (it == ranks.end()) it = ranks.emplace(max_pi, rank_cofactor_pis(dag, kMaxCofactorPis, max_pi)).first;
        std::vector<int32_t> pis(it->second.begin(), it->second.begin() + std::min<size_t>(k, it->second.size()));
        std::sort(pis.begin(), pis.end());
        return pis;
    }
    const LutNet &variant_set(const std::vector<int32_t> &pis, int copies = 0) {  // caller holds mu
        if (copies >= (1 << pis.size())) copies = 0;
        auto &slot = nets[{pis, copies}];
        if (!slot) {
            NvtxRange nvtx("es_map");
            slot.reset(new LutNet());
            std::vector<int32_t> ids;
            for (int c = 0; c < copies; ++c) ids.push_back(c);
            map_cofactored(dag, pis, slot.get(), copies ? &ids : nullptr);
        }
        return *slot;
    }
    const LutNet &variant(int k) { return variant_set(ranked(k)); }
    JitKernel *&jk(const LutNet &n, int threads) {
        return jks[{{n.cof_pis, (int)n.copy_ids.size()}, k1_slot(threads)}];
    }
};
// Hash of every program array, 8 bytes a step in four independent lanes (a
// warm call hashes mult16's 54 KB of arrays; byte-wise FNV-1a took ~70 us).
// A hit is confirmed against the stored arrays, so the hash only routes.
static uint64_t prog_hash(const es_prog &p) {
    uint64_t lane[4] = {0x9E3779B97F4A7C15ull, 0xC2B2AE3D27D4EB4Full, 0x165667B19E3779F9ull, 0x27D4EB2F165667C5ull};
    auto mix = [&](const void *d, size_t n) {
        const unsigned char *b = (const unsigned char *)d;
        size_t i = 0;
        for (; i + 32 <= n; i += 32)
            for (int q = 0; q < 4; ++q) {
                uint64_t w;
                std::memcpy(&w, b + i + 8 * q, 8);
                lane[q] = (lane[q] ^ w) * 0x9FB21C651E98DF25ull;
                lane[q] ^= lane[q] >> 29;
            }
        uint64_t t = n;
        for (; i < n; ++i) t = (t ^ b[i]) * 1099511628211ull;
        lane[0] = (lane[0] ^ t) * 0x9FB21C651E98DF25ull;
        lane[0] ^= lane[0] >> 29;
    };
    mix(&p.num_instrs, 4); mix(&p.num_registers, 4); mix(&p.num_pis, 4);
    const size_t n = (size_t)p.num_instrs;
    mix(p.op, n); mix(p.dst, 4 * n); mix(p.src0, 4 * n); mix(p.neg0, n);
    mix(p.src1, 4 * n); mix(p.neg1, n); mix(p.pi, 4 * n);
    uint64_t h = lane[0];
    for (int q = 1; q < 4; ++q) h = (h ^ lane[q]) * 0x9FB21C651E98DF25ull, h ^= h >> 31;
    return h;
}

// all program arrays, concatenated (the exact identity behind the hash key)
static std::vector<uint8_t> prog_sig(const es_prog &p) {
    const size_t n = (size_t)p.num_instrs;
    std::vector<uint8_t> v(12 + n * 19);
    uint8_t *d = v.data();
    auto put = [&](const void *s, size_t b) { std::memcpy(d, s, b); d += b; };
    put(&p.num_instrs, 4); put(&p.num_registers, 4); put(&p.num_pis, 4);
    put(p.op, n); put(p.dst, 4 * n); put(p.src0, 4 * n); put(p.neg0, n);
    put(p.src1, 4 * n); put(p.neg1, n); put(p.pi, 4 * n);
    return v;
}

// p's arrays equal a stored signature (compared in place, no copy)
static bool sig_equal(const es_prog &p, const std::vector<uint8_t> &sig) {
    const size_t n = (size_t)p.num_instrs;
    if (sig.size() != 12 + n * 19) return false;
    const uint8_t *d = sig.data();
    auto same = [&](const void *s, size_t b) {
        const bool e = std::memcmp(d, s, b) == 0;
        d += b;
        return e;
    };
    return same(&p.num_instrs, 4) && same(&p.num_registers, 4) && same(&p.num_pis, 4) && same(p.op, n) &&
           same(p.dst, 4 * n) && same(p.src0, 4 * n) && same(p.neg0, n) && same(p.src1, 4 * n) &&
           same(p.neg1, n) && same(p.pi, 4 * n);
}

static std::mutex g_mapped_mu;
static std::vector<std::pair<uint64_t, std::shared_ptr<MappedProg>>> g_mapped;

static int get_mapped(const es_prog &p, std::shared_ptr<MappedProg> *out) {
    const uint64_t key = prog_hash(p);
    {
        std::lock_guard<std::mutex> lk(g_mapped_mu);
        for (auto &kv : g_mapped)  // hash hit + identical arrays (no collision risk)
            if (kv.first == key && sig_equal(p, kv.second->sig)) { *out = kv.second; return ES_OK; }
    }
    std::vector<uint8_t> sig = prog_sig(p);
    Dag dag;
    std::string err;
    int rc = build_dag(p, &dag, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    auto mp = std::make_shared<MappedProg>();
    mp->sig = std::move(sig);
    mp->dag = std::move(dag);
    for (int i = 0; i < p.num_instrs; ++i) mp->G += (p.op[i] == ES_OP_AND || p.op[i] == ES_OP_XOR);
    std::lock_guard<std::mutex> lk(g_mapped_mu);
    if (g_mapped.size() >= 4096) g_mapped.clear();  // bound host memory for long sweeps
    g_mapped.push_back({key, mp});
    *out = mp;
    return ES_OK;
}

static bool constant_rail(const es_prog &p, es_result *r) {
    // es.py:265-270: OUTPUT reading the constant rail needs no sweep
    const int last = p.num_instrs - 1;
    if (p.src0[last] >= 0) return false;
    if (p.neg0[last]) {
        r->verdict = ES_COUNTEREXAMPLE;
        r->witness_index = 0;
        r->witness_minimal = 1;
        r->patterns_evaluated = 0;
    } else {
        r->verdict = ES_EXHAUSTED_ZERO;
        r->patterns_evaluated = 1ull << p.num_pis;
    }
    return true;
}

static int validate(const es_prog &p) {
    if (p.num_pis > ES_MAX_PIS) { set_error("too many inputs"); return ES_E_TOO_MANY_INPUTS; }
    if (p.num_pis < 0 || p.num_instrs < 1 || p.op[p.num_instrs - 1] != ES_OP_OUTPUT) {
        set_error("malformed program");
        return ES_E_BAD_PROGRAM;
    }
    return ES_OK;
}

// K1 cofactor depth (es_cofactor.cpp).  Estimates from round-1 B200
// measurements: ~1.9e13 LUT-words/s per 148 SMs for the sweep, ~0.1 ms of
// PTX->SASS per LUT for the JIT (mult16: 1,549 LUTs in 140 ms).
static double est_sweep_ms(const LutNet &n, int P, int sms) {
    const int k = (int)n.cof_pis.size();
    // beyond ~330 live values the kernel spills (255-register cap); fitted on
    // mult16: 358 live -> x1.12, 446 live (5 cofactor PIs) -> x2.6
    const double over = std::max(0.0, n.peak_live - 330.0);
    const double spill = 1.0 + 1.5e-4 * over * over;
    return 1e3 * spill * (double)n.luts.size() * std::ldexp(1.0, std::max(P - 5 - k, 0)) /
           (1.9e13 * sms / 148.0);
}
// ptxas time per LUT grows with register pressure (mult16 -O3: 0.09 ms/LUT
// at 143 live values, 0.15 at 212, 0.53 at 446); -O1 compiles in ~60 % of
// that (k=0: 95 vs 140 ms) for kernels 0.6-9 % slower
static double est_jit_ms(const LutNet &n, int opt = 3) {
    const double p = n.peak_live / 200.0;
    return (opt >= 3 ? 0.09 : 0.056) * std::max(1.0, p * p) * (double)n.luts.size();
}
constexpr double kO1Slowdown = 1.07;
// Direct SASS (es_sass.cpp): ~2 ms from LUT network to loaded module, the
// kernel slower than ptxas's by this factor (B200, mult16: k=0 12.0 vs 10.5 ms at
// -O1, k=4 2.69 vs 2.35 ms at -O3)
constexpr double kDirectJitMs = 2.0;
constexpr int kDirectMaxLive = 215;
static double direct_slowdown() {
    static const double v = getenv("ES_DIRECT_SLOW") ? atof(getenv("ES_DIRECT_SLOW")) : 1.15;
    return v;
}

// Split build (es_split.cpp, build level -P): ptxas on P phase modules in
// parallel host threads, then one nvJitLink.  Fitted on the B200 box (16
// host threads; mult16 k=0 / k=2, ES_JIT_CACHE=0): JIT = 0.75 * J1 / P +
// 40 ms + 0.4 ms * P (J1 = the one-body -O1 JIT; the constant is the link,
// module load and per-module ptxas start-up), and the sweep runs 1 + 0.09 P
// times the one-body kernel's time (shared-memory slot traffic at the cuts).
// mult16 k=0: J1 95 ms -> P=8 50 ms, sweep 10.5 -> 18.0 ms.
// es_run_opts.flags bit set by run_batch_jit: its jobs already compile on
// parallel host threads, so none of them may split (internal, not in the ABI)
constexpr int32_t kFlagNoSplit = 1 << 30;
static int split_parts(const LutNet &n, const es_run_opts &o) {
    if (o.flags & kFlagNoSplit) return 0;
    int P = o.jit_parts >= 2 ? o.jit_parts : 0;
    if (const char *e = getenv("ES_JIT_PARTS")) P = atoi(e);
    if (P == 0) P = (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
    if (P < 2 || (int)n.luts.size() < 16 * P) return 0;
    return P;
}
static double est_split_jit_ms(const LutNet &n, int P) {
    return 0.75 * est_jit_ms(n, 1) / P + 40.0 + 0.4 * P;
}
static double split_slowdown(int P) { return 1.0 + 0.09 * P; }

// ptxas level for variant k: throughput mode always -O3; otherwise the level
// with the smaller compile + expected sweep time (a kernel already compiled
// at that level or higher costs nothing), so a cold single run compiles at
// -O1 and a program that keeps being re-run tiers up to -O3.
static int k1_opt(const MappedProg &mp, const LutNet &n, const JitKernel *have, int P, int sms, bool tput,
                  double *cost, const es_run_opts &o) {
    const double sweep = est_sweep_ms(n, P, sms);
    const int parts = o.jit_parts == 1 ? 0 : split_parts(n, o);
    if (o.jit_parts >= 2 && parts >= 2) {  // forced split build
        *cost = (have && have->opt >= -parts ? 0.0 : est_split_jit_ms(n, parts)) + sweep * split_slowdown(parts);
        return -parts;
    }
    // direct SASS: a template for the variant and a live set that fits its
    // ~230 registers with the masks and coefficients (mult16 k=4: 212 LUT
    // values fit, k=5's 446 do not)
    const bool direct_ok = n.peak_live <= kDirectMaxLive && sass_template_exists(have ? have->block : o.block_threads > 0 ? o.block_threads
                                                     : n.cof_pis.empty() ? 128 : 256,
                                                 n.outs.size() > 1 || !n.cof_pis.empty());
    if (o.jit_parts == -1) {  // forced direct SASS (falls back to a ptxas build when it does not fit)
        *cost = (have ? 0.0 : kDirectJitMs) + sweep * direct_slowdown();
        return kJitDirect;
    }
    if (tput) { *cost = sweep; return 3; }
    const double reuse = 1.0 + mp.runs;  // doubling rule: expect as many more runs as so far
    // a batch compiles its jobs on every host thread while the device sweeps
    // earlier ones: a direct build (~1-3 ms) costs the device ~1/threads of
    // its time; a ptxas build (0.1-1 s) would still hold up the jobs queued
    // behind it, so a batch only takes one for a variant direct SASS cannot
    // hold, at its full cost
    const bool batch = (o.flags & kFlagNoSplit) != 0;
    const double jit_scale = batch ? 1.0 / std::max(1u, std::thread::hardware_concurrency()) : 1.0;
    int best = 3;
    *cost = 1e300;
    for (int opt : {3, 1, -parts, kJitDirect}) {
        if (opt == 0) continue;  // no split candidate
        if (opt == kJitDirect && (!direct_ok || o.jit_parts >= 1)) continue;
        if (batch && direct_ok && opt != kJitDirect && !(have && have->opt >= opt)) continue;
        const double jit = (have && have->opt >= opt) ? 0.0
                           : opt == kJitDirect ? jit_scale * kDirectJitMs
                           : opt < 0 ? est_split_jit_ms(n, parts) : est_jit_ms(n, opt);
        const double slow = opt == 3 ? 1.0 : opt == 1 ? kO1Slowdown
                            : opt == kJitDirect ? direct_slowdown() : kO1Slowdown * split_slowdown(parts);
        const double c = jit + sweep * reuse * slow;
        if (c < *cost) { *cost = c; best = opt; }
    }
    return best;
}

static int choose_cofactors(MappedProg &mp, const es_run_opts &o, int sms, int *opt) {
    const int P = mp.dag.num_pis;
    const bool tput = o.cofactor_pis == ES_COFACTOR_THROUGHPUT;
    double cost = 0;
    auto fixed = [&](int k) {
        const LutNet &n = mp.variant(k);
        *opt = k1_opt(mp, n, mp.jk(n, k1_threads(o, k)), P, sms, tput, &cost, o);
        return k;
    };
    if (o.cofactor_pis == ES_COFACTOR_NONE) return fixed(0);
    if (o.cofactor_pis > 0) {  // forced: any k the word PIs allow
        if (P - 5 < 1) return fixed(0);
        const LutNet &n = mp.variant(std::min(o.cofactor_pis, std::min(kMaxCofactorPis, P - 5)));
        return fixed((int)n.cof_pis.size());
    }
    // keep >= 2^14 kernel words so the grid still fills the GPU
    const int kmax = std::max(0, std::min(kMaxCofactorPis, P - 5 - 14));
    if (kmax == 0) return fixed(0);
    const LutNet &net0 = mp.variant(0);
    const double sweep0 = est_sweep_ms(net0, P, sms);
    // latency mode: a short sweep is JIT-bound; don't even map the variants
    // (not in a batch: its compiles and mappings overlap the device)
    const bool batch = (o.flags & kFlagNoSplit) != 0;
    if (!tput && !batch && sweep0 * (1 + mp.runs) < 0.1 * est_jit_ms(net0)) return fixed(0);
    int best = 0, worse = 0;
    double best_cost = 1e300, prev_cost = 0, map_ms = 0;
    for (int k = 0; k <= kmax; ++k) {
        const double tm = now_ms();
        const LutNet &n = mp.variant(k);
        const double this_map = now_ms() - tm;  // 0 when the variant was mapped before
        if ((int)n.cof_pis.size() != k) break;  // fewer candidate PIs than k
        const int ok = k1_opt(mp, n, mp.jk(n, k1_threads(o, k)), P, sms, tput, &cost, o);
        if (cost < best_cost) { best_cost = cost; best = k; *opt = ok; worse = 0; }
        // latency mode: the JIT term grows with k, so two deeper variants that
        // do not pay end the search (mapping k=3..5 costs ~40 ms on mult16)
        else if (!tput && ++worse >= 2) break;
        if (!tput && k > 0 && this_map > 0) {
            // mapping the next variant costs about twice this one (the
            // expansion doubles); stop when that exceeds what it can save
            // at the rate the last step saved (direct SASS makes the JIT
            // term flat, so host mapping time is what bounds the search).
            // A batch maps its jobs on every host thread while the device
            // sweeps: its mapping costs the device 1/threads of its time.
            map_ms = this_map * (batch ? 1.0 / std::max(1u, std::thread::hardware_concurrency()) : 1.0);
            const double gain = std::max(0.0, prev_cost - cost);
            if (2.0 * map_ms > 0.5 * gain) break;
        }
        prev_cost = cost;
    }
    return best;
}

// Compile-or-fetch the K1 kernel of variant `n` and plan its sweep over the
// devices of `cs` (chunk size for all of them).
static int k1_plan_for(MappedProg &mp, const LutNet &n, const es_run_opts &o, int sms, int n_dev, int opt,
                       K1Plan *pl, double *jit_ms) {
    const int threads = k1_threads(o, (int)n.cof_pis.size());
    JitKernel *&slot = mp.jk(n, threads);
    if (slot && slot->opt < opt) slot = nullptr;  // tier-up: recompile at the higher level (old module stays cached)
    int rc = k1_prepare(n, threads, sms, pl, jit_ms, slot, opt, n_dev);
    if (rc == ES_OK) slot = pl->jk;
    return rc;
}

// Fraction of a variant's kernel words whose first pattern (cofactor bits
// zero) is <= w: the part of the space a sweep with running minimum w must
// visit (first patterns are monotone in the word index: binary search).
static double frac_at_or_below(const std::vector<int32_t> &pis, int P, uint64_t w) {
    const int k = (int)pis.size();
    const int bits = std::max(P - 5 - k, 0);
    auto first = [&](uint64_t x) {
        x <<= 5;
        for (int32_t j : pis) {  // ascending pattern bits j-1
            const unsigned s = (unsigned)(j - 1);
            x = ((x >> s) << (s + 1)) | (x & ((1ull << s) - 1ull));
        }
        return x;
    };
    uint64_t lo = 0, hi = 1ull << bits;  // count of x with first(x) <= w, in [lo, hi]
    if (first(0) > w) return 0.0;
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (first(mid) <= w) lo = mid; else hi = mid;
    }
    return std::ldexp((double)(lo + 1), -bits);
}

// Whether variant `pl`'s chunks are contiguous pattern intervals: its
// cofactor bits all lie inside a chunk.  If not (the cheapest cofactor PIs
// are usually the top ones, e.g. the multiplier's b12..b15 = pattern bits
// 28..31), a chunk spans every value of those bits, and a counterexample
// above 2^28 leaves every chunk's first pattern below it: the skip rule can
// never fire (config 5 cost 1.03x the full EQ sweep).
static bool chunks_contiguous(const K1Plan &pl) {
    for (int i = 0; i < pl.cof_n; ++i)
        if ((int)pl.cof_pos[i] >= pl.chunk_log2 + 5 + pl.cof_n) return false;
    return true;
}

// K1 run of variant `net` on the devices `cs`, minimum-index witness for any
// cofactor set.  Non-contiguous chunks run in two phases:
//   1. the fast variant, stopping at the FIRST counterexample w1 (hit_stop);
//      if w1 lies below every chunk not yet swept, it is the minimum;
//   2. otherwise the cheaper of (a) finishing phase 1's sweep with w1 as the
//      running minimum, or (b) a variant whose cofactor PIs all lie below
//      w1's top bit, whose chunks are ordered like w1's high bits, so its
//      sweep stops after the ~w1/2^n of the space below w1.
// The minimum over both phases is the reference's workers=1 witness.
static int run_k1_job(MappedProg &mp, const LutNet &net, const es_run_opts &o, const std::vector<Ctx *> &cs,
                      double deadline, int opt, es_result *r) {
    NvtxRange nvtx("es_k1");
    const int n_dev = (int)cs.size();
    const int sms = cs[0]->sms;
    const int P = net.num_pis, G = mp.G;
    const uint64_t sentinel = 1ull << P;
    const bool tput = o.cofactor_pis == ES_COFACTOR_THROUGHPUT;
    K1Plan pl;
    double jit_ms = 0;
    int rc = k1_plan_for(mp, net, o, sms, n_dev, opt, &pl, &jit_ms);
    if (rc != ES_OK) return rc;
    r->engine = ES_ENGINE_JIT;
    r->jit_ms += jit_ms;
    r->regs_per_thread = pl.jk->regs;
    r->cofactor_pis = pl.cof_n;
    r->jit_opt = pl.jk->opt == kJitDirect ? 0 : pl.jk->opt < 0 ? 1 : pl.jk->opt;
    r->jit_parts = pl.jk->opt == kJitDirect ? -1 : pl.jk->parts;
    r->num_luts = (int)net.luts.size();
    r->n_devices = n_dev;
    r->phases = 1;
    const bool two_phase = !chunks_contiguous(pl);
    SweepOut s1;
    rc = sweep_k1(pl, G, o, cs, deadline, 0, sentinel, two_phase ? sentinel : 0, &s1);
    if (rc != ES_OK) return rc;
    const bool proven = s1.best < sentinel && (s1.prefix >= pl.n_chunks || s1.best < pl.first_pattern(s1.prefix));
    if (!two_phase || s1.stopped || s1.best >= sentinel || proven) {
        if (two_phase && s1.best >= sentinel && !s1.stopped && s1.prefix < pl.n_chunks) {
            // cannot happen: phase 1 only stops early on a hit
            set_error("internal: phase 1 ended early without a counterexample");
            return ES_E_CUDA;
        }
        k1_result(pl, s1, P, r);
        return ES_OK;
    }
    // phase 2
    r->phases = 2;
    const uint64_t w1 = s1.best;
    const double frac_left = 1.0 - (double)s1.prefix / (double)pl.n_chunks;
    const double cost_a = frac_left * est_sweep_ms(net, P, sms * n_dev);
    // the chunk holding w1: phase 1 may have left chunks below it unswept
    // (a claim that read the minimum after w1 landed skips its chunk)
    uint64_t cw1 = w1;  // w1 with its cofactor bits removed, in chunks
    for (int b = pl.cof_n - 1; b >= 0; --b) {
        const unsigned s = pl.cof_pos[b];
        cw1 = ((cw1 >> (s + 1)) << s) | (cw1 & ((1ull << s) - 1ull));
    }
    cw1 >>= pl.chunk_log2 + 5;
    // candidates: the cheapest PIs below one of w1's top set bits (PI j is
    // pattern bit j-1, so "PIs <= b" keeps every cofactor bit below bit b),
    // at the same depth or one less; cost = the exact fraction of the space
    // whose chunks start at or below w1, times the variant's sweep estimate
    std::vector<int> tops;
    for (int b = 63 - __builtin_clzll(w1); b >= kLanePis + 1 && tops.size() < 3; --b)
        if ((w1 >> b) & 1ull) tops.push_back(b);
    const LutNet *best_net = nullptr;
    double best_cost = cost_a;
    const int k0 = (int)net.cof_pis.size();
    for (int max_pi : tops)
        for (int k = k0; k >= std::max(0, k0 - 1); --k) {
            std::vector<int32_t> pis = mp.ranked(k, max_pi);
            if ((int)pis.size() != k) continue;
            const LutNet &cand = mp.variant_set(pis);
            double c = frac_at_or_below(pis, P, w1) * est_sweep_ms(cand, P, sms * n_dev);
            const JitKernel *have = mp.jk(cand, k1_threads(o, k));
            if (!tput && !(have && have->opt >= opt)) c += opt < 0 ? est_split_jit_ms(cand, -opt) : est_jit_ms(cand, opt);
            if (c < best_cost) { best_cost = c; best_net = &cand; }
        }
    // (c): the phase-1 cofactor set restricted to the copies below w1's copy c1
    // (a smaller body, same chunk order) over the chunks phase 1 left: every
    // pattern below w1 is either in a swept chunk or in one of those copies
    int c1 = 0;
    for (int b = 0; b < pl.cof_n; ++b) c1 |= (int)((w1 >> pl.cof_pos[b]) & 1ull) << b;
    const LutNet *restricted = nullptr;
    if (c1 > 0 && c1 < (1 << pl.cof_n)) {
        const LutNet &cand = mp.variant_set(net.cof_pis, c1);
        double c = frac_left * est_sweep_ms(cand, P, sms * n_dev);
        const JitKernel *have = mp.jk(cand, k1_threads(o, pl.cof_n));
        if (!tput && !(have && have->opt >= opt)) c += opt < 0 ? est_split_jit_ms(cand, -opt) : est_jit_ms(cand, opt);
        if (c < best_cost) { best_cost = c; best_net = nullptr; restricted = &cand; }
    }
    SweepOut s2;
    if (restricted) {
        K1Plan pl2;
        double jit2 = 0;
        rc = k1_plan_for(mp, *restricted, o, sms, n_dev, opt, &pl2, &jit2);
        if (rc != ES_OK) return rc;
        r->jit_ms += jit2;
        // every copy of the chunks phase 1 left below w1's (few: the claims in
        // flight when w1 landed), with the phase-1 variant
        SweepOut gap;
        gap.best = w1;
        if (s1.prefix <= cw1) {
            rc = sweep_k1(pl, G, o, cs, deadline, s1.prefix, w1, 0, &gap, cw1 + 1);
            if (rc != ES_OK) return rc;
            r->device_ms += gap.device_ms;
            r->launches += gap.launches;
            r->patterns_swept += gap.swept * pl.patterns_per_chunk();
        }
        // then copies 0..c1-1 of everything phase 1 left, in the restricted
        // plan's chunk units (rounded down)
        const uint64_t from = ((s1.prefix << pl.chunk_log2) >> pl2.chunk_log2);
        rc = sweep_k1(pl2, G, o, cs, deadline, from, gap.best, 0, &s2);
        if (rc != ES_OK) return rc;
        s2.stopped = s2.stopped || gap.stopped;
        s2.reason = s2.reason ? s2.reason : gap.reason;
        r->device_ms += s1.device_ms;
        r->launches += s1.launches;
        r->patterns_swept += std::min<uint64_t>(s1.swept * pl.patterns_per_chunk(), sentinel);
        r->phase2_cofactor_pis = pl2.cof_n;
        r->phase2_copies = c1;
        // the proof: phase 1 swept chunks [0, s1.prefix) of every copy, phase 2
        // copies [0, c1) of the rest; a stop leaves the prefix of both
        r->patterns_swept += (s2.swept << (pl2.chunk_log2 + 5)) * (uint64_t)c1;  // c1 copies per chunk word
        SweepOut s3 = s2;
        s3.swept = 0;
        s3.prefix = s2.stopped ? std::min(s1.prefix, (s2.prefix << pl2.chunk_log2) >> pl.chunk_log2) : pl.n_chunks;
        k1_result(pl, s3, P, r);
        return ES_OK;
    }
    if (!best_net) {  // (a): finish phase 1's sweep, skipping chunks above w1
        rc = sweep_k1(pl, G, o, cs, deadline, s1.prefix, w1, 0, &s2);
        if (rc != ES_OK) return rc;
        s2.swept += s1.swept;
        s2.device_ms += s1.device_ms;
        s2.launches += s1.launches;
        s2.prefix = s2.stopped ? std::min(s1.prefix, s2.prefix) : pl.n_chunks;
        k1_result(pl, s2, P, r);
        return ES_OK;
    }
    // (b): the low-cofactor variant over the space below w1
    K1Plan pl2;
    double jit2 = 0;
    rc = k1_plan_for(mp, *best_net, o, sms, n_dev, opt, &pl2, &jit2);
    if (rc != ES_OK) return rc;
    r->jit_ms += jit2;
    rc = sweep_k1(pl2, G, o, cs, deadline, 0, w1, 0, &s2);
    if (rc != ES_OK) return rc;
    r->device_ms += s1.device_ms;
    r->launches += s1.launches;
    r->patterns_swept += std::min<uint64_t>(s1.swept * pl.patterns_per_chunk(), sentinel);
    r->phase2_cofactor_pis = pl2.cof_n;
    k1_result(pl2, s2, P, r);
    return ES_OK;
}

int run_one(const es_prog *prog, const es_run_opts *opts, es_result *out) {
    NvtxRange nvtx("es_run");
    const double t0 = now_ms();
    std::memset(out, 0, sizeof(*out));
    es_run_opts o{};
    if (opts) o = *opts;
    int rc = validate(*prog);
    if (rc != ES_OK) return rc;
    const double deadline = o.budget_s >= 0 && opts ? t0 + 1e3 * o.budget_s : -1.0;
    if (constant_rail(*prog, out)) { out->wall_ms = now_ms() - t0; return ES_OK; }
    int reason = 0;
    if (stop_requested(o, deadline, &reason)) {  // es.py:299-309 before the first batch
        out->verdict = ES_BUDGET_EXCEEDED;
        out->reason = reason;
        out->wall_ms = now_ms() - t0;
        return ES_OK;
    }
    std::shared_ptr<MappedProg> mp;
    rc = get_mapped(*prog, &mp);
    if (rc != ES_OK) return rc;
    const int G = mp->G;
    out->compile_ms = now_ms() - t0;
    // one leased context per device of the run (the same ordinal may repeat)
    const std::vector<int> devs = run_devices(o);
    std::vector<std::unique_ptr<CtxLease>> leases;
    std::vector<Ctx *> cs;
    for (int d : devs) {
        leases.emplace_back(new CtxLease());
        rc = leases.back()->acquire(d);
        if (rc != ES_OK) return rc;
        cs.push_back(leases.back()->c);
    }
    Ctx *c = cs[0];
    out->n_devices = 1;
    int engine = o.engine;
    if (engine == ES_ENGINE_AUTO) {
        // The interpreter needs no JIT, the straight-line kernel sweeps ~40x
        // faster once compiled.  Estimates (B200 measurements): K2 ~5e13
        // gate-patterns/s (mult12: 2.5e10 in 0.45 ms), K1 ~2e15 plus ~0.02 ms
        // of launch; building K1 costs mapping (~1.2 us per gate: mult16 3.3
        // ms) plus the direct-SASS build (~1-2 ms; ptxas, 0.04 ms per gate at
        // -O1, only when the body does not fit a template).
        // Big sweeps go to K1; small ones to K1 when it is already compiled
        // or, in throughput mode, when its sweep is faster (JIT ignored);
        // otherwise by the doubling rule on the program's run count, so a
        // re-run program tiers up from K2 to K1 (mult12 at ~130 runs).
        const double work = (double)G * std::ldexp(1.0, prog->num_pis);
        const double k2_ms = 1e3 * work / 5e13, k1_ms = 0.02 + 1e3 * work / 2e15;
        bool compiled = false;
        double reuse = 1.0;
        {
            std::lock_guard<std::mutex> lk(mp->mu);
            for (const auto &kv : mp->jks) compiled = compiled || kv.second != nullptr;
            reuse += mp->runs + mp->k2_runs;
        }
        const bool tput = o.cofactor_pis == ES_COFACTOR_THROUGHPUT;
        const double jit_ms = compiled ? 0.0 : kDirectJitMs + 0.0012 * G;
        if (work >= 4e12) engine = ES_ENGINE_JIT;
        else if (tput || compiled) engine = k1_ms < k2_ms ? ES_ENGINE_JIT : ES_ENGINE_INTERP;
        else engine = jit_ms + k1_ms * reuse < k2_ms * reuse ? ES_ENGINE_JIT : ES_ENGINE_INTERP;
    }
    if (engine == ES_ENGINE_INTERP) {
        std::vector<int> act{0};
        const K2Prog *kp;
        std::shared_ptr<K2Prog> hold;  // a concurrent tier-up may replace mp->k2
        bool unfit = false;
        {
            std::lock_guard<std::mutex> lk(mp->mu);
            const double tc = now_ms();
            // one program: search cofactor depths when the sweep (~4 ms of
            // interpreter time and up) outweighs the host search, when the
            // caller asks for throughput, or once re-runs have paid for it
            const bool tput = o.cofactor_pis == ES_COFACTOR_THROUGHPUT;
            const double work = (double)G * std::ldexp(1.0, prog->num_pis);
            const bool tier_up = mp->k2 && !mp->k2_searched && (tput || work * (1 + mp->k2_runs) >= 2e11);
            if (!mp->k2 || tier_up) {
                const bool search = tput || work * (1 + mp->k2_runs) >= 2e11;
                auto fresh = std::make_shared<K2Prog>();
                build_k2prog_auto(mp->dag, fresh.get(), 9, 176, search ? 0.0 : 1e300);
                mp->k2 = fresh;
                mp->k2_searched = search;
            }
            mp->k2_runs++;
            hold = mp->k2;
            kp = hold.get();
            out->compile_ms += now_ms() - tc;
            unfit = !k2_fits(*kp);
        }
        if (!unfit) {
            rc = run_k2(1, prog, act, o, c, deadline, out, &kp);
        } else if (o.engine == ES_ENGINE_INTERP) {
            set_error("program needs " + std::to_string(kp->num_slots) + " slots (" +
                      std::to_string(k2_smem_w1(kp->num_slots, k2_device_records(*kp))) +
                      " B of shared memory): too many for the K2 interpreter; use engine auto or jit");
            return ES_E_BAD_PROGRAM;
        } else {
            engine = ES_ENGINE_JIT;  // auto: the live set is too wide for shared memory -> registers (K1)
        }
    }
    if (engine == ES_ENGINE_JIT) {
        std::lock_guard<std::mutex> lk(mp->mu);
        const double tc = now_ms();
        int opt = 3;
        // a batch job runs what its compile thread chose and built (searching
        // again here would find the variants mapped and pick anew, compiling
        // on this thread while the device waits)
        const bool prechosen = t_batch_jit && mp->batch_k >= 0;
        const int k = prechosen ? mp->batch_k : choose_cofactors(*mp, o, c->sms * (int)cs.size(), &opt);
        if (prechosen) opt = mp->batch_opt;
        mp->batch_k = -1;
        const LutNet &kn = mp->variant(k);
        out->compile_ms += now_ms() - tc;
        rc = run_k1_job(*mp, kn, o, cs, deadline, opt, out);
        mp->runs++;
        if (getenv("ES_VERBOSE"))
            fprintf(stderr, "[es] K1 run: %d PIs, %d gates, k=%d build %d, jit %.2f ms, device %.3f ms, %s\n",
                    prog->num_pis, G, k, opt, out->jit_ms, out->device_ms,
                    out->verdict == ES_EXHAUSTED_ZERO ? "EQ" : out->verdict == ES_COUNTEREXAMPLE ? "CEX" : "stop");
    }
    out->wall_ms = now_ms() - t0;
    return rc;
}

// Sub-miters as large as whole miters (a sweep's late-column pairs of a 16x16
// multiplier are 32-PI cones of ~2,800 gates) are K1 work: compile all their
// kernels on parallel host threads first (each is its own program), then run
// them one after another on the device.
int run_batch_jit(int n_jobs, const es_prog *progs, const es_run_opts *opts, es_result *outs) {
    NvtxRange nvtx("es_batch_k1");
    es_run_opts o{};
    if (opts) o = *opts;
    o.engine = ES_ENGINE_JIT;
    // the jobs already compile on parallel host threads: one-body ptxas builds,
    // or direct SASS where the policy prefers it, never split builds
    o.flags |= kFlagNoSplit;
    const double t0 = now_ms();
    const double deadline = o.budget_s >= 0 && opts ? t0 + 1e3 * o.budget_s : -1.0;
    int sms = 0;
    if (cudaGetDeviceCount(&sms) != cudaSuccess || sms == 0) { set_error("no CUDA device visible"); return ES_E_NO_DEVICE; }
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device));
    // compile on worker threads; run each job on this thread as soon as its
    // kernel is ready (in job order), so device sweeps overlap later compiles
    std::atomic<int> next{0};
    std::vector<uint8_t> ready(n_jobs, 0);
    std::mutex rmu;
    std::condition_variable rcv;
    auto mark = [&](int i) {
        { std::lock_guard<std::mutex> lk(rmu); ready[i] = 1; }
        rcv.notify_all();
    };
    auto warm = [&]() {
        t_batch_jit = true;
        const bool dev_ok = cudaSetDevice(o.device) == cudaSuccess;
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= n_jobs) return;
            if (dev_ok && validate(progs[i]) == ES_OK && progs[i].src0[progs[i].num_instrs - 1] >= 0) {
                std::shared_ptr<MappedProg> mp;
                if (get_mapped(progs[i], &mp) == ES_OK) {
                    std::lock_guard<std::mutex> lk(mp->mu);
                    int opt = 3;
                    const int k = choose_cofactors(*mp, o, sms * (int)run_devices(o).size(), &opt);
                    mp->batch_k = k;  // the run on the main thread uses this decision
                    mp->batch_opt = opt;
                    const LutNet &net = mp->variant(k);
                    const int threads = k1_threads(o, k);
                    JitKernel *&have = mp->jk(net, threads);
                    if (!(have && have->opt >= opt)) {
                        JitKernel *jk = nullptr;
                        double ms = 0;
                        std::string err;
                        if (jit_get(net, threads, &jk, &ms, &err, opt) == ES_OK) have = jk;
                    }
                }
            }
            mark(i);  // failures surface in run_one
        }
    };
    const int nt = (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), (unsigned)n_jobs);
    std::vector<std::thread> th;
    for (int q = 0; q < nt; ++q) th.emplace_back(warm);
    int rc = ES_OK;
    for (int i = 0; i < n_jobs && rc == ES_OK; ++i) {
        {
            std::unique_lock<std::mutex> lk(rmu);
            rcv.wait(lk, [&] { return ready[i] != 0; });
        }
        es_run_opts oi = o;
        if (deadline >= 0) oi.budget_s = std::max(0.0, (deadline - now_ms()) * 1e-3);
        t_batch_jit = true;
        rc = run_one(&progs[i], &oi, &outs[i]);
        t_batch_jit = false;
    }
    next.store(n_jobs);  // on an error, stop compiling what will not run
    for (auto &x : th) x.join();
    if (getenv("ES_VERBOSE"))
        fprintf(stderr, "[es batch k1] jobs=%d compile threads=%d wall=%.2fms\n", n_jobs, nt, now_ms() - t0);
    return rc;
}

int run_batch(int n_jobs, const es_prog *progs, const es_run_opts *opts, es_result *outs,
              const K2Prog *const *prebuilt) {
    const double t0 = now_ms();
    es_run_opts o{};
    if (opts) o = *opts;
    const double deadline = o.budget_s >= 0 && opts ? t0 + 1e3 * o.budget_s : -1.0;
    std::vector<int> active;
    for (int j = 0; j < n_jobs; ++j) {
        std::memset(&outs[j], 0, sizeof(es_result));
        // batch sub-miters were compiled and checked (build_dag) at extraction
        int rc = prebuilt ? ES_OK : validate(progs[j]);
        if (rc != ES_OK) return rc;
        if (!constant_rail(progs[j], &outs[j])) active.push_back(j);
    }
    if (active.empty()) return ES_OK;
    CtxLease lease;
    int rc = lease.acquire(o.device);
    if (rc != ES_OK) return rc;
    Ctx *c = lease.c;
    int reason = 0;
    if (stop_requested(o, deadline, &reason)) {
        for (int j : active) { outs[j].verdict = ES_BUDGET_EXCEEDED; outs[j].reason = reason; }
        return ES_OK;
    }
    std::vector<int> unfit;
    rc = run_k2(n_jobs, progs, active, o, c, deadline, outs, prebuilt,
                o.engine == ES_ENGINE_INTERP ? nullptr : &unfit);
    // live sets too wide for the interpreter's shared memory run on K1
    for (size_t q = 0; q < unfit.size() && rc == ES_OK; ++q) {
        es_run_opts oj = o;
        oj.engine = ES_ENGINE_JIT;
        if (deadline >= 0) oj.budget_s = std::max(0.0, (deadline - now_ms()) * 1e-3);
        rc = run_one(&progs[unfit[q]], &oj, &outs[unfit[q]]);
    }
    const double wall = now_ms() - t0;
    for (int j = 0; j < n_jobs; ++j) outs[j].wall_ms = wall;
    return rc;
}

// ---------------------------------------------------------------------------
// sessions (multi-GPU sharding through the caller's collectives)
// ---------------------------------------------------------------------------
struct Session {
    int dev = 0;
    K1Plan plan;
    LutNet net;
    unsigned *d_counter = nullptr;
    int num_pis = 0;
};

int session_open(const es_prog *prog, const es_run_opts *opts, void **out) {
    es_run_opts o{};
    if (opts) o = *opts;
    int rc = validate(*prog);
    if (rc != ES_OK) return rc;
    if (prog->src0[prog->num_instrs - 1] < 0) { set_error("constant-rail program: nothing to sweep"); return ES_E_BAD_ARG; }
    Dag dag;
    std::string err;
    rc = build_dag(*prog, &dag, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    CtxLease lease;
    rc = lease.acquire(o.device);
    if (rc != ES_OK) return rc;
    Ctx *c = lease.c;
    Session *s = new Session();
    s->dev = o.device;
    s->num_pis = prog->num_pis;
    int opt = 3;
    {
        std::shared_ptr<MappedProg> mp;
        rc = get_mapped(*prog, &mp);
        if (rc != ES_OK) { delete s; return rc; }
        std::lock_guard<std::mutex> lk(mp->mu);
        s->net = mp->variant(choose_cofactors(*mp, o, c->sms, &opt));
    }
    double jit_ms = 0;
    rc = k1_prepare(s->net, k1_threads(o, (int)s->net.cof_pis.size()), c->sms, &s->plan, &jit_ms,
                    nullptr, opt);
    if (rc != ES_OK) { delete s; return rc; }
    if (cudaMalloc(&s->d_counter, 64) != cudaSuccess) { delete s; set_error("cudaMalloc"); return ES_E_CUDA; }
    *out = s;
    return ES_OK;
}

int session_geometry(const void *sp, uint64_t *n_chunks, uint64_t *ppc, int32_t *luts, int32_t *regs) {
    const Session *s = (const Session *)sp;
    if (n_chunks) *n_chunks = s->plan.n_chunks;
    if (ppc) *ppc = s->plan.patterns_per_chunk();
    if (luts) *luts = (int32_t)s->net.luts.size();
    if (regs) *regs = s->plan.jk->regs;
    return ES_OK;
}

int session_launch(void *sp, void *stream, uint64_t *best_dev, uint64_t chunk_begin,
                   uint64_t chunk_end, int rank, int world) {
    Session *s = (Session *)sp;
    if (world < 1 || rank < 0 || rank >= world || chunk_end < chunk_begin) { set_error("bad shard"); return ES_E_BAD_ARG; }
    CK(cudaSetDevice(s->dev));
    chunk_end = std::min<uint64_t>(chunk_end, s->plan.n_chunks);
    if (chunk_begin >= chunk_end) return ES_OK;
    const uint64_t W = (uint64_t)world;
    const uint64_t first = chunk_begin + ((uint64_t)rank + W - chunk_begin % W) % W;
    if (first >= chunk_end) return ES_OK;
    const uint64_t n_slots = (chunk_end - first + W - 1) / W;
    return k1_launch(s->plan, (cudaStream_t)stream, (unsigned long long *)best_dev, s->d_counter,
                     first, n_slots, W);
}

void session_close(void *sp) {
    Session *s = (Session *)sp;
    if (!s) return;
    cudaSetDevice(s->dev);
    if (s->d_counter) cudaFree(s->d_counter);
    delete s;
}

int fma_peak(int dev, double *lane_ops_per_s, double *ms_out) {
    CtxLease lease;
    int rc = lease.acquire(dev);
    if (rc != ES_OK) return rc;
    Ctx *c = lease.c;
    const int threads = 256, iters = 2048;
    const int grid = c->sms * 8;
    unsigned *sink = c->d_counter + 8;
    es_imad_peak_kernel<<<grid, threads, 0, c->stream>>>(sink, 64, 1u);  // warm-up
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_start, c->stream));
    es_imad_peak_kernel<<<grid, threads, 0, c->stream>>>(sink, iters, 1u);
    CK(cudaEventRecord(c->ev_stop, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev_start, c->ev_stop));
    *lane_ops_per_s = (double)grid * threads * (double)iters * 64.0 / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    return ES_OK;
}

int alu_peak(int dev, double *lane_ops_per_s, double *ms_out) {
    CtxLease lease;
    int rc = lease.acquire(dev);
    if (rc != ES_OK) return rc;
    Ctx *c = lease.c;
    const int threads = 256, iters = 4096;
    const int grid = c->sms * 8;
    unsigned *sink = c->d_counter + 8;
    es_alu_peak_kernel<<<grid, threads, 0, c->stream>>>(sink, 64, 1u);  // warm-up
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_start, c->stream));
    es_alu_peak_kernel<<<grid, threads, 0, c->stream>>>(sink, iters, 1u);
    CK(cudaEventRecord(c->ev_stop, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev_start, c->ev_stop));
    const double ops = (double)grid * threads * (double)iters * 64.0;
    *lane_ops_per_s = ops / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    return ES_OK;
}

int smem_peak(int dev, double *bytes_per_s, double *ms_out) {
    CtxLease lease;
    int rc = lease.acquire(dev);
    if (rc != ES_OK) return rc;
    Ctx *c = lease.c;
    const int threads = 256, iters = 2048;
    const int grid = c->sms * 8;
    unsigned *sink = c->d_counter + 8;
    es_smem_peak_kernel<<<grid, threads, 0, c->stream>>>(sink, 32);  // warm-up
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_start, c->stream));
    es_smem_peak_kernel<<<grid, threads, 0, c->stream>>>(sink, iters);
    CK(cudaEventRecord(c->ev_stop, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev_start, c->ev_stop));
    *bytes_per_s = (double)grid * threads * (double)iters * 8.0 * 16.0 / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    return ES_OK;
}

// ---------------------------------------------------------------------------
// cross-process shared minimum word (CUDA IPC; NVLink peer memory across GPUs)
// ---------------------------------------------------------------------------
// Layout of one exchange slot: [0] the minimum word, [8] the arrival counter.
// Device-side verdict barrier: after its sweep kernel (same stream), every
// rank's es_peer_arrive adds one to the counter with system scope, waits
// until all `world` ranks have arrived, then copies the final minimum to
// `out` -- no host round trip and no collective between verdicts, so the
// host can queue verdict after verdict.  Rank 0 re-arms the slot two
// verdicts ahead (es_peer_arm): every rank has passed that slot's barrier
// before rank 0 can pass the previous one.
__global__ void es_peer_arm_kernel(unsigned long long *word) {
    word[0] = ~0ull;
    reinterpret_cast<unsigned *>(word + 1)[0] = 0u;
    __threadfence_system();
}

__global__ void es_peer_arrive_kernel(unsigned long long *word, unsigned world, unsigned long long *out) {
    unsigned *counter = reinterpret_cast<unsigned *>(word + 1);
    __threadfence_system();  // this rank's sweep (stream-ordered before us) is complete
    atomicAdd_system(counter, 1u);
    unsigned v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        if (v >= world) break;
        __nanosleep(100);
    }
    unsigned long long w;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(word) : "memory");
    *out = w;
}

int peer_arm(void *stream, void *word) {
    es_peer_arm_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long *)word);
    CK(cudaGetLastError());
    return ES_OK;
}

int peer_arrive_wait(void *stream, void *word, int world, void *out) {
    if (world < 1) { set_error("bad world size"); return ES_E_BAD_ARG; }
    es_peer_arrive_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((unsigned long long *)word, (unsigned)world,
                                                            (unsigned long long *)out);
    CK(cudaGetLastError());
    return ES_OK;
}

int ipc_alloc(int dev, void **ptr, unsigned char *handle) {
    CK(cudaSetDevice(dev));
    CK(cudaMalloc(ptr, 256));
    CK(cudaMemset(*ptr, 0, 256));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, *ptr));
    memcpy(handle, &h, sizeof(h));
    return ES_OK;
}

int ipc_open(int dev, const unsigned char *handle, void **ptr) {
    CK(cudaSetDevice(dev));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return ES_OK;
}

int ipc_close(int dev, void *ptr, int owner) {
    CK(cudaSetDevice(dev));
    if (owner) { CK(cudaFree(ptr)); }
    else { CK(cudaIpcCloseMemHandle(ptr)); }
    return ES_OK;
}

int word_io(int dev, void *ptr, uint64_t *value, int write) {
    CK(cudaSetDevice(dev));
    if (write) { CK(cudaMemcpy(ptr, value, 8, cudaMemcpyHostToDevice)); }
    else { CK(cudaMemcpy(value, ptr, 8, cudaMemcpyDeviceToHost)); }
    return ES_OK;
}

void runtime_shutdown() {
    {
        std::lock_guard<std::mutex> lk(g_k4_mu);
        for (auto &kv : g_k4_mods) {
            for (K4Img &x : kv.second->imgs) cudaFree(x.d_img);
            cudaLibraryUnload(kv.second->lib);
        }
        g_k4_mods.clear();
    }
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (Ctx *c : g_ctx_all) {
        cudaSetDevice(c->dev);
        cudaStreamDestroy(c->stream);
        cudaFree(c->d_best);
        cudaFree(c->d_counter);
        cudaFreeHost(c->h_pin);
        if (c->h_stage) cudaFreeHost(c->h_stage);
        cudaEventDestroy(c->ev_start);
        cudaEventDestroy(c->ev_stop);
        cudaEventDestroy(c->ev_slice[0]);
        cudaEventDestroy(c->ev_slice[1]);
        for (int q = 0; q < 7; ++q) {
            cudaStreamDestroy(c->side[q]);
            cudaEventDestroy(c->ev_side[q]);
        }
        delete c;
    }
    g_ctx_all.clear();
    g_ctx_free.clear();
    {
        std::lock_guard<std::mutex> lk(g_mapped_mu);
        g_mapped.clear();
    }
    jit_clear();
}

}  // namespace es
