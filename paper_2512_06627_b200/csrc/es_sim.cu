// es_sim.cu -- K3: word-parallel random simulation of a whole XAG (sm_100a).
//
// Reference: cecprove/sim.py:21-38 (simulate) -- every node gets a row of
// 64-bit words, bit b of word w = the node's value under pattern 64*w+b --
// and sweep.py:54-81 (_signatures / build_pe_classes): nodes grouped by their
// polarity-canonical row.  SURVEY 8(f) next-3: the sweep's random simulation,
// candidate-class discovery and counterexample refinement.
//
// Layout in HBM is the reference's array: vals[node][word] (uint64,
// row-major), PI rows = the caller's pi_words, node 0 = 0.  One thread per
// 64-bit word walks the gates level by level, in batches of up to kSimU
// gates of one level: it issues all 2*kSimU fanin loads of a batch (rows of
// earlier levels, L2-resident: the kernel sweeps the word space in tiles so
// the live rows of a tile fit in L2), then computes and stores the batch --
// loads and stores coalesced across the warp.  Every node row is written
// exactly once, so the kernel is bound by HBM writes: 8 bytes per gate per
// word (the drive and the fanin re-reads come from L2).
//
// Classes: one warp per node hashes its polarity-canonical row (polarity =
// bit 7 of word 0: the reference compares the rows' little-endian bytes, and
// the first byte of a row and of its complement always differ); the host
// groups nodes by hash, the device then checks every member's row against its
// group leader word by word, and only a failed check (a 64-bit collision)
// falls back to comparing downloaded rows on the host.  Classes are therefore
// exactly the reference's.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <tuple>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/es_b200.h"
#include "es_nvtx.h"

namespace es {

void set_error(const std::string &m);

namespace {

#define SCK(call)                                                                   \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));          \
            return ES_E_CUDA;                                                       \
        }                                                                           \
    } while (0)

// record: {fanin node a, fanin node b, output node, flags}; flags bit 0 XOR,
// 1 NEG_A, 2 NEG_B.  Gates are sorted by level and cut into batches of
// kSimU gates of one level (padded with flags bit 3: no-op).
struct SimRec {
    uint32_t a, b, d, f;
};
constexpr int kSimU = 16;  // measured (mult16, 65,536 words): 8 -> 0.57 ms, 16 -> 0.54, 32 -> 0.78

// G threads per word (lanes of one warp): thread g of a word evaluates gates
// g, g+G, ... of each batch, so G x more warps hide the latency of the
// sequential level chain; __syncwarp orders a batch's row stores before the
// next batch's loads (rows of one word are only touched by its G lanes).
template <int G>
__global__ void __launch_bounds__(256) es_sim_kernel(const SimRec *__restrict__ recs, int n_batches,
                                                     long long w_begin, long long w_end,
                                                     long long words,
                                                     unsigned long long *__restrict__ vals) {
    constexpr int U = kSimU / G;
    const int gi = threadIdx.x % G;
    const long long w = w_begin + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const bool active = w < w_end;
    if (__all_sync(0xffffffffu, !active)) return;
    for (int bt = 0; bt < n_batches; ++bt) {
        const SimRec *rb = recs + bt * kSimU + gi;
        unsigned long long x[U], y[U];
        SimRec r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = rb[u * G];
        if (active) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                x[u] = vals[(long long)r[u].a * words + w];
                y[u] = vals[(long long)r[u].b * words + w];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (r[u].f & 8u) continue;
                const unsigned long long xa = (r[u].f & 2u) ? ~x[u] : x[u];
                const unsigned long long yb = (r[u].f & 4u) ? ~y[u] : y[u];
                vals[(long long)r[u].d * words + w] = (r[u].f & 1u) ? (xa ^ yb) : (xa & yb);
            }
        }
        if (G > 1) __syncwarp();
    }
}

// Software-pipelined variant (SimProg::pipe): the host schedules batches so
// that batch t+1 reads no row written by batch t (every fanin was stored two
// or more batches earlier), so each thread issues batch t+1's fanin loads
// before it computes and stores batch t -- two batches' loads in flight, one
// round trip per two batches on the level chain instead of one per batch.
template <int G>
__global__ void __launch_bounds__(256) es_sim_pipe_kernel(const SimRec *__restrict__ recs, int n_batches,
                                                          long long w_begin, long long w_end,
                                                          long long words,
                                                          unsigned long long *__restrict__ vals) {
    constexpr int U = kSimU / G;
    const int gi = threadIdx.x % G;
    const long long w = w_begin + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const bool active = w < w_end;
    if (__all_sync(0xffffffffu, !active) || n_batches <= 0) return;
    unsigned long long x[U], y[U];
    uint32_t d[U], f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const SimRec r = recs[gi + u * G];
        d[u] = r.d; f[u] = r.f;
        x[u] = active ? vals[(long long)r.a * words + w] : 0ull;
        y[u] = active ? vals[(long long)r.b * words + w] : 0ull;
    }
    for (int bt = 0; bt < n_batches; ++bt) {
        unsigned long long nx[U], ny[U];
        uint32_t nd[U], nf[U];
        const bool more = bt + 1 < n_batches;
        const SimRec *rb = recs + (more ? bt + 1 : bt) * kSimU + gi;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const SimRec r = rb[u * G];
            nd[u] = r.d; nf[u] = r.f;
            nx[u] = (active && more) ? vals[(long long)r.a * words + w] : 0ull;
            ny[u] = (active && more) ? vals[(long long)r.b * words + w] : 0ull;
        }
        if (active) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (f[u] & 8u) continue;
                const unsigned long long xa = (f[u] & 2u) ? ~x[u] : x[u];
                const unsigned long long yb = (f[u] & 4u) ? ~y[u] : y[u];
                vals[(long long)d[u] * words + w] = (f[u] & 1u) ? (xa ^ yb) : (xa & yb);
            }
        }
        if (G > 1) __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u) { x[u] = nx[u]; y[u] = ny[u]; d[u] = nd[u]; f[u] = nf[u]; }
    }
}

// per node: polarity (bit 7 of word 0) and a 64-bit hash of the canonical row
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__global__ void es_sig_kernel(const unsigned long long *__restrict__ vals, int n_nodes, long long words,
                              unsigned long long *__restrict__ hash, unsigned char *__restrict__ pol) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n_nodes) return;
    const unsigned long long *row = vals + (long long)warp * words;
    const unsigned long long inv = (row[0] >> 7) & 1ull ? ~0ull : 0ull;
    unsigned long long h = 0;
    for (long long q = lane; q < words; q += 32)
        h += mix64((row[q] ^ inv) + 0x9e3779b97f4a7c15ull * (unsigned long long)(q + 1));
#pragma unroll
    for (int off = 16; off; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
    if (lane == 0) {
        hash[warp] = mix64(h ^ (unsigned long long)words);
        pol[warp] = (unsigned char)(inv & 1ull);
    }
}

// per-node count of 1-bits over all simulated patterns (ones_fraction,
// sim.py:45-48), one warp per node row: only the counts leave the device
__global__ void es_ones_kernel(const unsigned long long *__restrict__ vals, int n_nodes, long long words,
                               long long *__restrict__ counts) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n_nodes) return;
    const unsigned long long *row = vals + (long long)warp * words;
    long long c = 0;
    for (long long q = lane; q < words; q += 32) c += __popcll(row[q]);
#pragma unroll
    for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (lane == 0) counts[warp] = c;
}

// members[i] vs leader[i]: canonical rows equal?  one warp per pair
__global__ void es_verify_kernel(const unsigned long long *__restrict__ vals, long long words,
                                 const int *__restrict__ member, const int *__restrict__ leader, int n,
                                 const unsigned char *__restrict__ pol, int *__restrict__ bad) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int m = member[warp], l = leader[warp];
    const unsigned long long im = pol[m] ? ~0ull : 0ull, il = pol[l] ? ~0ull : 0ull;
    const unsigned long long *rm = vals + (long long)m * words, *rl = vals + (long long)l * words;
    int diff = 0;
    for (long long q = lane; q < words; q += 32) diff |= (rm[q] ^ im) != (rl[q] ^ il);
    diff = __any_sync(0xffffffffu, diff);
    if (lane == 0) bad[warp] = diff;
}

struct SimProg {
    std::vector<SimRec> recs;  // whole batches: the level schedule, then the distance-2 one
    int levels = 0;
    size_t n_level = 0;  // records of the level schedule (es_sim_kernel)
};

// Distance-2 list schedule (appended after the level batches): a gate may go into batch t once
// both fanins were written in batches <= t-2 (PIs/constant: always); up to
// kSimU ready gates per batch, longest path to a sink first.
void schedule_pipe(int FG, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                   const uint32_t *in1, SimProg *sp) {
    constexpr int D = 2;
    const int NG = num_gates;
    std::vector<int> fo_start(NG + 1, 0), fo(2 * (size_t)NG), pend(NG, 0), height(NG, 0), bidx(NG, 0);
    for (int g = 0; g < NG; ++g)
        for (uint32_t l : {in0[g], in1[g]}) {
            const int a = (int)(l >> 1) - FG;
            if (a >= 0) { fo_start[a + 1]++; pend[g]++; }
        }
    for (int g = 0; g < NG; ++g) fo_start[g + 1] += fo_start[g];
    {
        std::vector<int> fill(fo_start.begin(), fo_start.end() - 1);
        for (int g = 0; g < NG; ++g)
            for (uint32_t l : {in0[g], in1[g]}) {
                const int a = (int)(l >> 1) - FG;
                if (a >= 0) fo[fill[a]++] = g;
            }
    }
    for (int g = NG - 1; g >= 0; --g)
        for (uint32_t l : {in0[g], in1[g]}) {
            const int a = (int)(l >> 1) - FG;
            if (a >= 0) height[a] = std::max(height[a], height[g] + 1);
        }
    std::vector<std::vector<int>> bucket(1);
    for (int g = 0; g < NG; ++g)
        if (pend[g] == 0) bucket[0].push_back(g);
    std::priority_queue<std::pair<int, int>> ready;  // (height, -gate)
    int placed = 0;
    for (int t = 0; placed < NG; ++t) {
        if ((int)bucket.size() > t)
            for (int g : bucket[t]) ready.push({height[g], -g});
        std::vector<int> batch;
        while (!ready.empty() && (int)batch.size() < kSimU) {
            batch.push_back(-ready.top().second);
            ready.pop();
        }
        for (int g : batch) {
            bidx[g] = t;
            SimRec r{};
            r.a = in0[g] >> 1;
            r.b = in1[g] >> 1;
            r.d = (uint32_t)(FG + g);
            r.f = (kind[g] ? 1u : 0u) | ((in0[g] & 1) ? 2u : 0u) | ((in1[g] & 1) ? 4u : 0u);
            sp->recs.push_back(r);
        }
        placed += (int)batch.size();
        for (int g : batch)
            for (int e = fo_start[g]; e < fo_start[g + 1]; ++e) {
                const int o = fo[e];
                if (--pend[o]) continue;
                int rt = 0;
                for (uint32_t l : {in0[o], in1[o]}) {
                    const int a = (int)(l >> 1) - FG;
                    if (a >= 0) rt = std::max(rt, bidx[a] + D);
                }
                if ((int)bucket.size() <= rt) bucket.resize(rt + 1);
                bucket[rt].push_back(o);
            }
        // an empty batch still occupies batch index t (the distance rule counts batches)
        if (batch.empty()) sp->recs.push_back(SimRec{0, 0, 0, 8u});
        while (sp->recs.size() % kSimU) sp->recs.push_back(SimRec{0, 0, 0, 8u});
    }
}

// Levelised gate list: level(v) = 1 + max level of its gate fanins; gates
// sorted by (level, node), each level cut into batches of kSimU (the last
// batch of a level padded with no-ops), so a batch never reads a row it
// writes.
int build_sim_prog(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                   const uint32_t *in1, SimProg *sp) {
    const int FG = 1 + num_pis, NN = FG + num_gates;
    std::vector<int> lvl(NN, 0);
    int max_lvl = 0;
    for (int g = 0; g < num_gates; ++g) {
        const int v = FG + g, a = (int)(in0[g] >> 1), b = (int)(in1[g] >> 1);
        if (a >= v || b >= v) { set_error("simulation: XAG not topological"); return ES_E_BAD_PROGRAM; }
        lvl[v] = 1 + std::max(lvl[a], lvl[b]);
        max_lvl = std::max(max_lvl, lvl[v]);
    }
    std::vector<int> start(max_lvl + 2, 0), order(num_gates);
    for (int g = 0; g < num_gates; ++g) start[lvl[FG + g] + 1]++;
    for (int l = 0; l <= max_lvl; ++l) start[l + 1] += start[l];
    {
        std::vector<int> fill(start.begin(), start.end() - 1);
        for (int g = 0; g < num_gates; ++g) order[fill[lvl[FG + g]]++] = g;
    }
    sp->recs.clear();
    sp->levels = max_lvl;
    for (int l = 1; l <= max_lvl; ++l) {
        for (int q = start[l]; q < start[l + 1]; ++q) {
            const int g = order[q];
            SimRec r{};
            r.a = in0[g] >> 1;
            r.b = in1[g] >> 1;
            r.d = (uint32_t)(FG + g);
            r.f = (kind[g] ? 1u : 0u) | ((in0[g] & 1) ? 2u : 0u) | ((in1[g] & 1) ? 4u : 0u);
            sp->recs.push_back(r);
        }
        while (sp->recs.size() % kSimU) sp->recs.push_back(SimRec{0, 0, 0, 8u});
    }
    sp->n_level = sp->recs.size();
    schedule_pipe(FG, num_gates, kind, in0, in1, sp);
    return ES_OK;
}

struct SimDev {
    int dev = -1;
    cudaStream_t st = nullptr;
};

int sim_device(int dev, SimDev **out) {
    static thread_local std::vector<SimDev *> ctx;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) { set_error("no CUDA device visible"); return ES_E_NO_DEVICE; }
    if (dev < 0 || dev >= n) { set_error("device ordinal out of range"); return ES_E_BAD_ARG; }
    SCK(cudaSetDevice(dev));
    for (SimDev *c : ctx)
        if (c->dev == dev) { *out = c; return ES_OK; }
    SimDev *c = new SimDev();
    c->dev = dev;
    SCK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    cudaMemPool_t pool;  // keep freed per-call buffers cached (see es_runtime.cu:get_ctx)
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    ctx.push_back(c);
    *out = c;
    return ES_OK;
}

// Enqueue the simulation on `st` with device buffers (vals: num_nodes x words).
// The word space is swept in tiles whose live rows fit in L2 (the fanin
// re-reads then never reach HBM).
int sim_enqueue(const SimProg &sp, const SimRec *d_recs, int num_pis, long long words,
                const unsigned long long *d_pi, unsigned long long *d_vals, cudaStream_t st,
                long long num_nodes) {
    SCK(cudaMemsetAsync(d_vals, 0, (size_t)words * 8, st));  // node 0 = 0
    if (num_pis > 0)
        SCK(cudaMemcpyAsync(d_vals + words, d_pi, (size_t)num_pis * words * 8, cudaMemcpyDeviceToDevice, st));
    if (sp.recs.empty()) return ES_OK;
    const int T = 256;
    // tile: all rows of the tile <= ~48 MB (a third of L2), >= 2 waves of CTAs
    long long tile = std::max<long long>(T * 148 * 2, (48ll << 20) / (8 * std::max<long long>(num_nodes, 1)));
    tile = (tile + T - 1) / T * T;
    for (long long w0 = 0; w0 < words; w0 += tile) {
        const long long w1 = std::min(words, w0 + tile);
        // threads per word: the level chain is latency-bound, so small drives
        // (the sweep's 64 words) take more lanes per word.  mult16, us, for
        // G = 1/2/4/8: 64 words ~300/166/138/113; 8,192: -/-/202/182;
        // 16,384: 375/272/227/309; 32,768: 390/317/372/-; 65,536: 535/584/720/-
        const long long nw = w1 - w0;
        int G = nw <= 8192 ? 8 : nw <= 16384 ? 4 : nw <= 32768 ? 2 : 1;
        if (const char *e = getenv("ES_SIM_G")) G = atoi(e);
        const long long grid = (nw * G + T - 1) / T;
        // software-pipelined kernel for tiles of <= 16,384 words (mult16, us,
        // level / pipelined at the default G: 64 words 112/109, 4,096: 154/147,
        // 16,384: 227/204; 65,536 words (G = 1): 532/840, G = 2 647)
        bool pipe = nw <= 16384;
        if (const char *e = getenv("ES_SIM_PIPE")) pipe = atoi(e) != 0;
        const int nb = (int)((pipe ? sp.recs.size() - sp.n_level : sp.n_level) / kSimU);
        if (pipe) {
            const SimRec *pr = d_recs + sp.n_level;
            if (G == 8) es_sim_pipe_kernel<8><<<(unsigned)grid, T, 0, st>>>(pr, nb, w0, w1, words, d_vals);
            else if (G == 4) es_sim_pipe_kernel<4><<<(unsigned)grid, T, 0, st>>>(pr, nb, w0, w1, words, d_vals);
            else if (G == 2) es_sim_pipe_kernel<2><<<(unsigned)grid, T, 0, st>>>(pr, nb, w0, w1, words, d_vals);
            else es_sim_pipe_kernel<1><<<(unsigned)grid, T, 0, st>>>(pr, nb, w0, w1, words, d_vals);
        } else if (G == 8) es_sim_kernel<8><<<(unsigned)grid, T, 0, st>>>(d_recs, nb, w0, w1, words, d_vals);
        else if (G == 4) es_sim_kernel<4><<<(unsigned)grid, T, 0, st>>>(d_recs, nb, w0, w1, words, d_vals);
        else if (G == 2) es_sim_kernel<2><<<(unsigned)grid, T, 0, st>>>(d_recs, nb, w0, w1, words, d_vals);
        else es_sim_kernel<1><<<(unsigned)grid, T, 0, st>>>(d_recs, nb, w0, w1, words, d_vals);
        SCK(cudaGetLastError());
    }
    return ES_OK;
}

}  // namespace

int sim_levels(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
              const uint32_t *in1) {
    SimProg sp;
    const int rc = build_sim_prog(num_pis, num_gates, kind, in0, in1, &sp);
    return rc == ES_OK ? sp.levels : rc;
}

// simulate() with host buffers (sim.py:21-38): node_words = num_nodes x words,
// and/or ones = per-node 1-bit counts (num_nodes int64)
static int sim_run_host(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                        const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
                        uint64_t *node_words, int64_t *ones, double *device_ms) {
    NvtxRange nvtx("es_sim");
    if (words < 1 || num_pis < 0 || num_gates < 0) { set_error("bad argument"); return ES_E_BAD_ARG; }
    SimProg sp;
    int rc = build_sim_prog(num_pis, num_gates, kind, in0, in1, &sp);
    if (rc != ES_OK) return rc;
    SimDev *c = nullptr;
    rc = sim_device(device, &c);
    if (rc != ES_OK) return rc;
    const long long NN = 1 + num_pis + num_gates;
    SimRec *d_recs = nullptr;
    unsigned long long *d_pi = nullptr, *d_vals = nullptr;
    SCK(cudaMallocAsync(&d_recs, std::max<size_t>(sp.recs.size(), 1) * sizeof(SimRec), c->st));
    SCK(cudaMallocAsync(&d_pi, std::max<size_t>((size_t)num_pis * words, 1) * 8, c->st));
    long long *d_ones = nullptr;
    SCK(cudaMallocAsync(&d_vals, (size_t)NN * words * 8, c->st));
    if (ones) SCK(cudaMallocAsync(&d_ones, (size_t)NN * 8, c->st));
    if (!sp.recs.empty())
        SCK(cudaMemcpyAsync(d_recs, sp.recs.data(), sp.recs.size() * sizeof(SimRec), cudaMemcpyHostToDevice, c->st));
    if (num_pis > 0)
        SCK(cudaMemcpyAsync(d_pi, pi_words, (size_t)num_pis * words * 8, cudaMemcpyHostToDevice, c->st));
    cudaEvent_t e0, e1;
    SCK(cudaEventCreate(&e0));
    SCK(cudaEventCreate(&e1));
    SCK(cudaEventRecord(e0, c->st));
    rc = sim_enqueue(sp, d_recs, num_pis, words, d_pi, d_vals, c->st, NN);
    if (rc == ES_OK && ones) {
        es_ones_kernel<<<(unsigned)((NN * 32 + 255) / 256), 256, 0, c->st>>>(d_vals, (int)NN, words, d_ones);
        SCK(cudaGetLastError());
    }
    SCK(cudaEventRecord(e1, c->st));
    if (rc == ES_OK && node_words)
        SCK(cudaMemcpyAsync(node_words, d_vals, (size_t)NN * words * 8, cudaMemcpyDeviceToHost, c->st));
    if (rc == ES_OK && ones)
        SCK(cudaMemcpyAsync(ones, d_ones, (size_t)NN * 8, cudaMemcpyDeviceToHost, c->st));
    SCK(cudaStreamSynchronize(c->st));
    if (d_ones) cudaFreeAsync(d_ones, c->st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(d_recs, c->st);
    cudaFreeAsync(d_pi, c->st);
    cudaFreeAsync(d_vals, c->st);
    SCK(cudaStreamSynchronize(c->st));
    return rc;
}

int sim_run(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
            const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
            uint64_t *node_words, double *device_ms) {
    return sim_run_host(num_pis, num_gates, kind, in0, in1, pi_words, words, device, node_words, nullptr,
                        device_ms);
}

int sim_ones(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
             const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
             int64_t *ones, double *device_ms) {
    if (!ones) { set_error("bad argument"); return ES_E_BAD_ARG; }
    return sim_run_host(num_pis, num_gates, kind, in0, in1, pi_words, words, device, nullptr, ones,
                        device_ms);
}

// Device-resident variant for callers that own the buffers (torch tensors):
// enqueued on `stream`, no host synchronisation.
int sim_run_device(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                   const uint32_t *in1, const uint64_t *d_pi_words, int64_t words, void *stream,
                   uint64_t *d_node_words, void **prog_cache) {
    if (words < 1 || num_pis < 0 || num_gates < 0) { set_error("bad argument"); return ES_E_BAD_ARG; }
    struct Cached { SimProg sp; SimRec *d_recs = nullptr; };
    Cached *cp = prog_cache ? (Cached *)*prog_cache : nullptr;
    if (!cp) {
        cp = new Cached();
        int rc = build_sim_prog(num_pis, num_gates, kind, in0, in1, &cp->sp);
        if (rc != ES_OK) { delete cp; return rc; }
        SCK(cudaMalloc(&cp->d_recs, std::max<size_t>(cp->sp.recs.size(), 1) * sizeof(SimRec)));
        if (!cp->sp.recs.empty())
            SCK(cudaMemcpy(cp->d_recs, cp->sp.recs.data(), cp->sp.recs.size() * sizeof(SimRec), cudaMemcpyHostToDevice));
        if (prog_cache) *prog_cache = cp;
    }
    int rc = sim_enqueue(cp->sp, cp->d_recs, num_pis, words, (const unsigned long long *)d_pi_words,
                         (unsigned long long *)d_node_words, (cudaStream_t)stream,
                         1ll + num_pis + num_gates);
    if (!prog_cache) {
        cudaStreamSynchronize((cudaStream_t)stream);
        cudaFree(cp->d_recs);
        delete cp;
    }
    return rc;
}

void sim_prog_free(void *prog_cache) {
    struct Cached { SimProg sp; SimRec *d_recs = nullptr; };
    Cached *cp = (Cached *)prog_cache;
    if (!cp) return;
    cudaFree(cp->d_recs);
    delete cp;
}

// random_simulate + build_pe_classes (sweep.py:66-81) from a PI drive:
// class_id[node] = index of its class in representative order, -1 for a
// singleton; polarity[node] = canonical polarity (inv < raw).
int sim_classes(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
                int32_t *class_id, uint8_t *polarity, int32_t *n_classes, double *device_ms) {
    NvtxRange nvtx("es_sim_classes");
    if (words < 1 || num_pis < 0 || num_gates < 0 || !class_id || !polarity || !n_classes) {
        set_error("bad argument");
        return ES_E_BAD_ARG;
    }
    SimProg sp;
    int rc = build_sim_prog(num_pis, num_gates, kind, in0, in1, &sp);
    if (rc != ES_OK) return rc;
    SimDev *c = nullptr;
    rc = sim_device(device, &c);
    if (rc != ES_OK) return rc;
    const int NN = 1 + num_pis + num_gates;
    SimRec *d_recs = nullptr;
    unsigned long long *d_pi = nullptr, *d_vals = nullptr, *d_hash = nullptr;
    unsigned char *d_pol = nullptr;
    SCK(cudaMallocAsync(&d_recs, std::max<size_t>(sp.recs.size(), 1) * sizeof(SimRec), c->st));
    SCK(cudaMallocAsync(&d_pi, std::max<size_t>((size_t)num_pis * words, 1) * 8, c->st));
    SCK(cudaMallocAsync(&d_vals, (size_t)NN * words * 8, c->st));
    SCK(cudaMallocAsync(&d_hash, (size_t)NN * 8, c->st));
    SCK(cudaMallocAsync(&d_pol, (size_t)NN, c->st));
    if (!sp.recs.empty())
        SCK(cudaMemcpyAsync(d_recs, sp.recs.data(), sp.recs.size() * sizeof(SimRec), cudaMemcpyHostToDevice, c->st));
    if (num_pis > 0)
        SCK(cudaMemcpyAsync(d_pi, pi_words, (size_t)num_pis * words * 8, cudaMemcpyHostToDevice, c->st));
    cudaEvent_t e0, e1;
    SCK(cudaEventCreate(&e0));
    SCK(cudaEventCreate(&e1));
    SCK(cudaEventRecord(e0, c->st));
    rc = sim_enqueue(sp, d_recs, num_pis, words, d_pi, d_vals, c->st, NN);
    if (rc != ES_OK) return rc;
    es_sig_kernel<<<(NN * 32 + 255) / 256, 256, 0, c->st>>>(d_vals, NN, words, d_hash, d_pol);
    SCK(cudaGetLastError());
    std::vector<unsigned long long> h(NN);
    std::vector<unsigned char> pol(NN);
    SCK(cudaMemcpyAsync(h.data(), d_hash, (size_t)NN * 8, cudaMemcpyDeviceToHost, c->st));
    SCK(cudaMemcpyAsync(pol.data(), d_pol, (size_t)NN, cudaMemcpyDeviceToHost, c->st));
    SCK(cudaStreamSynchronize(c->st));
    // group by hash; groups in first-member order = representative order
    std::unordered_map<unsigned long long, int> gid;
    gid.reserve((size_t)NN * 2);
    std::vector<int> group(NN), gsize, gleader;
    for (int v = 0; v < NN; ++v) {
        auto it = gid.find(h[v]);
        int g;
        if (it == gid.end()) { g = (int)gsize.size(); gid.emplace(h[v], g); gsize.push_back(0); gleader.push_back(v); }
        else g = it->second;
        group[v] = g;
        gsize[g]++;
    }
    // verify every non-leader member of a multi-node group on the device
    std::vector<int> mem, lead;
    for (int v = 0; v < NN; ++v)
        if (gsize[group[v]] >= 2 && gleader[group[v]] != v) { mem.push_back(v); lead.push_back(gleader[group[v]]); }
    std::vector<int> bad(mem.size(), 0);
    if (!mem.empty()) {
        int *d_m = nullptr, *d_l = nullptr, *d_bad = nullptr;
        const size_t nb = mem.size() * sizeof(int);
        SCK(cudaMallocAsync(&d_m, nb, c->st));
        SCK(cudaMallocAsync(&d_l, nb, c->st));
        SCK(cudaMallocAsync(&d_bad, nb, c->st));
        SCK(cudaMemcpyAsync(d_m, mem.data(), nb, cudaMemcpyHostToDevice, c->st));
        SCK(cudaMemcpyAsync(d_l, lead.data(), nb, cudaMemcpyHostToDevice, c->st));
        es_verify_kernel<<<(unsigned)((mem.size() * 32 + 255) / 256), 256, 0, c->st>>>(
            d_vals, words, d_m, d_l, (int)mem.size(), d_pol, d_bad);
        SCK(cudaGetLastError());
        SCK(cudaMemcpyAsync(bad.data(), d_bad, nb, cudaMemcpyDeviceToHost, c->st));
        SCK(cudaEventRecord(e1, c->st));
        SCK(cudaStreamSynchronize(c->st));
        cudaFreeAsync(d_m, c->st);
        cudaFreeAsync(d_l, c->st);
        cudaFreeAsync(d_bad, c->st);
    } else {
        SCK(cudaEventRecord(e1, c->st));
        SCK(cudaStreamSynchronize(c->st));
    }
    // a 64-bit collision: regroup that hash group exactly from downloaded rows
    std::vector<int> sub(NN, 0);  // sub-group within a hash group (0 = leader's)
    std::vector<char> split(gsize.size(), 0);
    for (size_t q = 0; q < mem.size(); ++q)
        if (bad[q]) split[group[mem[q]]] = 1;
    for (size_t g = 0; g < gsize.size(); ++g) {
        if (!split[g]) continue;
        std::vector<int> nodes;
        for (int v = 0; v < NN; ++v) if (group[v] == (int)g) nodes.push_back(v);
        std::vector<std::vector<unsigned long long>> rows(nodes.size(), std::vector<unsigned long long>(words));
        for (size_t q = 0; q < nodes.size(); ++q) {
            SCK(cudaMemcpy(rows[q].data(), d_vals + (long long)nodes[q] * words, words * 8, cudaMemcpyDeviceToHost));
            if (pol[nodes[q]]) for (auto &x : rows[q]) x = ~x;
        }
        int next = 0;
        std::vector<int> lab(nodes.size(), -1);
        for (size_t q = 0; q < nodes.size(); ++q) {
            if (lab[q] >= 0) continue;
            lab[q] = next++;
            for (size_t r = q + 1; r < nodes.size(); ++r)
                if (lab[r] < 0 && rows[r] == rows[q]) lab[r] = lab[q];
        }
        for (size_t q = 0; q < nodes.size(); ++q) sub[nodes[q]] = lab[q];
    }
    // class ids in representative (= first member) order, singletons -1
    std::unordered_map<long long, int> cid;
    std::unordered_map<long long, int> csize;
    for (int v = 0; v < NN; ++v) csize[(long long)group[v] * NN + sub[v]]++;
    int nc = 0;
    for (int v = 0; v < NN; ++v) {
        const long long key = (long long)group[v] * NN + sub[v];
        polarity[v] = pol[v];
        if (csize[key] < 2) { class_id[v] = -1; continue; }
        auto it = cid.find(key);
        if (it == cid.end()) { cid.emplace(key, nc); class_id[v] = nc++; }
        else class_id[v] = it->second;
    }
    *n_classes = nc;
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(d_recs, c->st);
    cudaFreeAsync(d_pi, c->st);
    cudaFreeAsync(d_vals, c->st);
    cudaFreeAsync(d_hash, c->st);
    cudaFreeAsync(d_pol, c->st);
    SCK(cudaStreamSynchronize(c->st));
    return ES_OK;
}

}  // namespace es
