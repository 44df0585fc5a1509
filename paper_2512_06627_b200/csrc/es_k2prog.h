// es_k2prog.h -- K2 interpreter program (internal).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "es_core.h"

namespace es {

// Record flags (K2Gate::ctl, low byte) and the copy number of an OUT record
// (ctl >> 16).
enum : uint32_t {
    K2_XOR = 1u,      // gate: A ^ B ^ ma (else (A ^ ma) & (B ^ mb))
    K2_A_ACC = 2u,    // operand A (gate) / the output value (OUT) is the accumulator
    K2_STORE = 8u,    // gate: store the result into slot d
    K2_OUT = 16u,     // output record: fold (A ^ ma) into (first failing word, copy)
    K2_NEG_A = 32u,   // ma = ~0
    K2_NEG_B = 64u,   // mb = ~0
    K2_CONST = 128u,  // OUT: the value is the constant 0 (then NEG_A makes it ~0)
};
// OUT with K2_A_ACC in a multi-lane program: the accumulator's lane (2 bits)
constexpr unsigned K2_OUT_LANE_SHIFT = 8;
constexpr int kK2MaxCofactorPis = 6;

// One 16-byte record: a gate or an output.  Slots on the host, byte offsets
// in the device image.
struct K2Gate {
    uint32_t a, b, d;  // operand / destination slot
    uint32_t ctl;      // K2_* flags | copy << 16
};
static_assert(sizeof(K2Gate) == 16, "K2Gate is the 16-byte device record");

// K4 body of a job (es_sass.cpp k4_body): the job's direct-SASS code for the
// K4 multi-body skeleton, built once per program and kept with it.
struct K4Body {
    std::vector<uint64_t> code;  // encoded instructions, (lo, hi) pairs
    uint64_t hash = 0;           // of `code` (module cache key)
    int instrs = 0;
    int variant = 0;             // K4 template variant (es_jit.h k4_blocks)
    bool ok = false;             // false: no body (too many registers / slots)
};

struct K2Prog {
    int num_pis = 0;
    int num_slots = 0;              // PI slots + gate slots
    std::vector<K2Gate> gates;      // gates and OUT records, in execution order
    std::vector<int32_t> cof_pis;   // cofactor PIs (ascending); copies = 2^size
    int n_gates = 0;                // gate records (excluding OUT)
    int loads = 0, stores = 0;      // slot loads / stores per pass (cost model)
    // Multi-lane program (lanes L = 2 or 4; kernel es_k2d): records come in
    // steps of L -- L independent gates, one per lane, each lane with its own
    // accumulator (a NOP lane is acc & ~0 over the zero slot num_pis), or up
    // to L OUT records (the rest NOPs).  Every lane's operands are read
    // before any result of the step is stored.
    int lanes = 1;
    mutable std::shared_ptr<K4Body> k4;  // built on demand by a batch run (run_k2)
};

// Launch group of a program: the widest words-per-thread W (4, 2, 1) at which
// its slot file (slots x 128 threads x W x 4 B) plus its staged records fit
// two CTAs per SM (2 x (bytes + 1 KB) <= 228 KB); 0 = W4, 1 = W2, 2 = W1.
constexpr size_t kK2TwoCtaBytes = 115600;
// records staged past a program's end (the kernels prefetch one step ahead)
constexpr int kK2PadRecords = 8;  // two steps of up to four lanes
inline int k2_group_of(int num_slots, size_t num_records) {
    const size_t rec = (num_records + kK2PadRecords) * 16, s = (size_t)(num_slots > 0 ? num_slots : 1) * 512;
    if (s * 4 + rec <= kK2TwoCtaBytes) return 0;
    if (s * 2 + rec <= kK2TwoCtaBytes) return 1;
    return 2;
}

// Whether the interpreter can run a program at all: its slot file at one word
// per thread plus its staged records (and the kernel's 16 static bytes) in
// one CTA's dynamic shared memory (B200 opt-in maximum, 227 KB).  Programs
// that do not fit go to K1 (es_runtime.cu routes them).
constexpr size_t kK2MaxSmemBytes = 232448 - 64;
inline size_t k2_smem_w1(int num_slots, size_t num_records) {
    return (size_t)(num_slots > 0 ? num_slots : 1) * 512 + (num_records + kK2PadRecords) * 16;
}
// Device records of a program (one per record).
inline size_t k2_device_records(const K2Prog &kp) { return kp.gates.size(); }
inline bool k2_fits(const K2Prog &kp) { return k2_smem_w1(kp.num_slots, k2_device_records(kp)) <= kK2MaxSmemBytes; }

// Lanes of the K2 programs build_k2prog emits (ES_K2_LANES: 1, 2 or 4).
int k2_lanes();
// K2 program of a (possibly multi-output) graph: DFS schedule with
// accumulator forwarding, LIFO slot reuse, OUT records in copy order.
void build_k2prog(const Dag &dag, K2Prog *kp);
// Pick the cofactor depth k (0..kK2MaxCofactorPis) that minimises the
// shared-memory traffic per word, keeping >= 2^min_words_log2 kernel words
// per job and <= max_slots slots (the interpreter's shared-memory limit at
// one word per thread); then build that program.  A sweep of fewer than
// min_work gate-patterns is not worth the host time of the search (k = 0).
void build_k2prog_auto(const Dag &dag, K2Prog *kp, int min_words_log2 = 9, int max_slots = 176,
                       double min_work = 0.0);
// Forced depth k (tests): the k word PIs of smallest fanout.
void build_k2prog_k(const Dag &dag, int k, K2Prog *kp);
// CPU model of the interpreter over FULL word indices [w0, w0+nw) (cofactor
// PIs included): each word's output is its copy's.
void eval_k2prog(const K2Prog &kp, uint64_t w0, uint64_t nw, uint32_t *out);

}  // namespace es
