// es_k2prog.h -- K2 interpreter program (internal).
#pragma once

#include <cstdint>
#include <vector>

#include "es_core.h"

namespace es {

enum : uint32_t { K2_XOR = 1u, K2_A_ACC = 2u, K2_B_ACC = 4u, K2_STORE = 8u };

// One gate of a K2 program: slots (host) or byte offsets (device image).
struct K2Gate {
    uint32_t a, b, d;  // operand / destination slot
    uint32_t ma, mb;   // complement masks (XOR: ma = both, mb = 0)
    uint32_t ctl;      // K2_* flags
};
static_assert(sizeof(K2Gate) == 24, "K2Gate is the 24-byte device record");

struct K2Prog {
    int num_pis = 0;
    int num_slots = 0;  // PI slots + gate slots
    uint32_t out_mask = 0;
    bool const_out = false;
    std::vector<K2Gate> gates;
};

void build_k2prog(const Dag &dag, K2Prog *kp);
// CPU model of the interpreter over words [w0, w0+nw) (kernel word layout).
void eval_k2prog(const K2Prog &kp, uint64_t w0, uint64_t nw, uint32_t *out);

}  // namespace es
