// es_core.h -- internal IR of the B200 ES engine (not part of the C ABI).
//
// Pipeline (host, C++):
//   es_prog (reference InstrProgram, es.py:66-73)
//     -> Dag        SSA graph rebuilt from the register program
//     -> LutNet     LUT-3 cover (one LOP3 per LUT), constant-folded low PIs
//     -> schedule   register-pressure-aware topological order
//     -> PTX body   spliced into the hand-written K1 skeleton (k1_skeleton.cu)
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/es_b200.h"

namespace es {

// Run fn(0..n-1) on all host cores (one thread per `grain` items at most:
// 256 for cheap items, 1 for items of a millisecond, e.g. K4 bodies).
template <class F>
inline void parallel_for(int n, F fn, int grain = 256) {
    const int nt = (int)std::min<int>(std::max(1u, std::thread::hardware_concurrency()),
                                      std::max(1, n / std::max(1, grain)));
    std::atomic<int> next{0};
    auto work = [&]() {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= n) return;
            fn(i);
        }
    };
    std::vector<std::thread> th;
    for (int q = 1; q < nt; ++q) th.emplace_back(work);
    work();
    for (auto &x : th) x.join();
}

// Pattern layout shared by every engine (kernel, CPU model, witness decode):
// pattern p = 32*w + b.  Bit b of a 32-bit word carries PIs 1..5
// (PI j = bit j-1 of b), the word index w carries PIs 6.. (PI j = bit j-6 of
// w).  This is the reference's pattern numbering (es.py:315-320) with 32-bit
// instead of 64-bit words.
constexpr int kWordBits = 32;
constexpr int kLanePis = 5;
extern const uint32_t kLaneMask[kLanePis];  // 0xAAAAAAAA, 0xCCCCCCCC, ...

// Node ids: 0 = constant FALSE, 1..num_pis = PIs, then gates.
struct Dag {
    int num_pis = 0;
    std::vector<uint8_t> is_xor;     // per gate
    std::vector<int32_t> f0, f1;     // fanin node ids, per gate
    std::vector<uint8_t> n0, n1;     // fanin complement flags, per gate
    int32_t out_node = 0;
    bool out_neg = false;
    // Multi-output graphs (cofactor expansion, es_cofactor.cpp): when `outs`
    // is non-empty it replaces (out_node, out_neg); output c is the miter
    // output under cofactor assignment c.
    std::vector<int32_t> outs;
    std::vector<uint8_t> outs_neg;
    int num_nodes() const { return 1 + num_pis + (int)is_xor.size(); }
    int first_gate() const { return 1 + num_pis; }
    bool is_pi(int v) const { return v >= 1 && v <= num_pis; }
};

// Rebuild the SSA graph from a reference register program.  Returns ES_OK or
// ES_E_BAD_PROGRAM (undefined source register, missing/extra OUTPUT, ...).
int build_dag(const es_prog &p, Dag *dag, std::string *err);

// One LUT: out = f(leaf0, leaf1, leaf2); tt bit i = f at leaf_k = bit k of i
// (so PTX `lop3.b32 d, leaf2, leaf1, leaf0, tt` computes it).  Leaves are
// node ids; a leaf is a PI, a folded constant, or another LUT.
struct Lut {
    int32_t node;
    int32_t leaf[3];
    uint8_t nleaves;
    uint8_t tt;
};

struct LutNet {
    int num_pis = 0;
    std::vector<Lut> luts;                // in schedule order (topological)
    std::vector<uint8_t> is_const;        // per node: value is a compile-time word
    std::vector<uint32_t> const_val;      // per node (valid when is_const)
    // output: either a LUT/PI/constant node with optional inversion folded in
    int32_t out_node = 0;
    bool out_neg = false;                 // inversion still to apply (only when out is a leaf)
    // all outputs, one per cofactor copy (outs[0] == out_node); 1 without cofactoring
    std::vector<int32_t> outs;
    std::vector<uint8_t> outs_neg;
    // Cofactor PIs (ascending, all >= 6): their values are fixed per copy, not
    // per word, so the kernel's word index w' enumerates the other PIs only.
    // pi_bit[j] = bit of w' carrying PI j (-1 for lane PIs 1..5 and cofactor PIs).
    std::vector<int32_t> cof_pis;
    std::vector<int8_t> pi_bit;
    // copy_ids[i] = the cofactor assignment of outs[i] (bit b = value of
    // cof_pis[b]); empty = all 2^k copies in order.  A restricted variant
    // evaluates only some copies (the second phase of a non-equivalent
    // search needs only the copies below the first witness's).
    std::vector<int32_t> copy_ids;
    int copy_id(size_t i) const { return copy_ids.empty() ? (int)i : copy_ids[i]; }
    int num_gates = 0;                    // AND+XOR gates in the output cone
    int peak_live = 0;                    // max simultaneously live LUT values in the schedule
    std::vector<int32_t> pis_used;        // PIs >= 6 referenced as leaves
};

// LUT-3 technology mapping (priority cuts + area flow + exact-area recovery)
// followed by a live-range-minimising schedule.
// Multi-output graphs map every output; cof_pis/pi_bit are left for the
// caller (default: no cofactors, pi_bit[j] = j - 6).
void map_luts(const Dag &dag, LutNet *net);

// Cofactor expansion (es_cofactor.cpp).  A PI that is fixed per copy is a
// constant inside each copy, so the logic in its transitive fanout folds;
// logic outside it is shared by all copies (structural hashing).  One kernel
// iteration then evaluates 2^k words -- one per assignment of the k cofactor
// PIs -- for the price of the shared logic once plus the folded copies.
constexpr int kMaxCofactorPis = 5;
// Rank word PIs (>= 6) by transitive-fanout size (cheapest first) and return
// the first `k` of that order (rank order: sort before cofactor_expand).
// max_pi: only PIs <= max_pi are candidates (the second phase of a
// non-equivalent sweep keeps its cofactor bits below the witness's top bit).
std::vector<int32_t> rank_cofactor_pis(const Dag &dag, int k, int max_pi = 1 << 20);
// dag with the PIs in `pis` (ascending) cofactored: 2^k outputs, output c
// under PI pis[b] = bit b of c.  Constant propagation + structural hashing.
// copies: the assignments to expand (ascending; nullptr = all 2^k).
void cofactor_expand(const Dag &dag, const std::vector<int32_t> &pis, Dag *out,
                     const std::vector<int32_t> *copies = nullptr);
// map_luts of the expansion, with cof_pis / pi_bit (and copy_ids) filled in.
void map_cofactored(const Dag &dag, const std::vector<int32_t> &pis, LutNet *net,
                    const std::vector<int32_t> *copies = nullptr);

// Reference compile_program (es.py:87-163), exact.
int32_t ref_compile(int32_t num_pis, int32_t num_gates, const uint8_t *kind,
                    const uint32_t *in0, const uint32_t *in1, uint32_t out_lit,
                    int8_t *op, int32_t *dst, int32_t *src0, uint8_t *neg0,
                    int32_t *src1, uint8_t *neg1, int32_t *pi, int32_t *num_registers);

// CPU model of the LUT program over words [w0, w0+nw): bit-exact with K1.
void eval_lutnet(const LutNet &net, uint64_t w0, uint64_t nw, uint32_t *out);

// PTX body for the K1 skeleton: reads the word index from (wlo, whi) and
// writes the output word to `out` (register names from the skeleton).
// `one` names a register holding 1 that ptxas cannot constant-fold; with it,
// LUTs of the form f(x, word PI) become FMA-pipe IMADs (empty: LOP3 only).
// Without cofactors `outs` = {output word}; with them {first failing copy's
// word (0: none), that copy's number} -- the K1 multi skeleton's operands.
std::string emit_body_ptx(const LutNet &net, const std::vector<std::string> &outs,
                          const std::string &wlo, const std::string &whi,
                          const std::string &one = "");

// A LUT that is a 2-input function of a word-uniform selector u and one
// other value x, as x*S + T (one FMA-pipe IMAD; es_compile.cpp).
struct ImadPlan {
    int x = -1, u = -1;  // node ids
    int s0, s1, t0, t1;  // x*S+T coefficients for u = 0 / u = 1
};
// sel[v]: v is word-uniform (a PI >= 6 or a LUT over such nodes).
bool plan_imad(const Lut &L, const std::vector<uint8_t> &sel, ImadPlan *pl);

// Shared-memory overflow slots for the K1 body (es_spill.cpp): rewrite a
// body from emit_body_ptx so that at most `budget` %es values are live in
// registers anywhere in the schedule (Belady eviction); evicted values are
// stored once (at the first eviction) to a per-thread slot of the dynamic
// shared array es_slots (slot s of thread t at (s*threads + t)*4) and
// reloaded before later uses.  Returns the body unchanged (slots 0) when
// nothing has to move.
struct SpillStats {
    int slots = 0;   // shared-memory words per thread
    int loads = 0;   // ld.shared per iteration
    int stores = 0;  // st.shared per iteration
    int peak = 0;    // register-resident values at the peak (<= budget)
};
std::string spill_body(const std::string &body, int budget, int threads, SpillStats *st);

// Split build of the K1 body (es_split.cpp): the LUT sequence cut into
// `parts` phases, each one a separately compiled PTX module holding one
// device function, so ptxas runs on the phases in parallel and the linker
// joins them.  Values live across a cut pass through per-thread shared-memory
// slots (slot s of thread t at es_slots + (s*threads + t)*4).
struct SplitPtx {
    std::vector<std::string> phases;  // complete PTX modules, one .func each
    std::string decls;                // module-scope .extern declarations for the caller
    std::string call_body;            // replaces the K1 skeleton's ES_BODY line
    int slots = 0;                    // shared-memory slots per thread
    int crossings = 0;                // values stored to a slot (one store each)
    int loads = 0;                    // slot loads over all phases (per iteration)
    std::vector<int> cuts;            // first LUT of each phase
};
bool emit_split_ptx(const LutNet &net, int threads, int parts, const std::string &header,
                    const std::vector<std::string> &outs, const std::string &wlo,
                    const std::string &whi, const std::string &one, SplitPtx *out);

uint32_t lane_valid_mask(int num_pis);

}  // namespace es
