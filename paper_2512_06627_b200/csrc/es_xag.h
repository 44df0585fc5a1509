// es_xag.h -- the reference's XAG builder in C++ (internal).
//
// cecprove/xag.py:128-192 (XagBuilder): the same structural-hashing key
// (kind, lo.pack(), hi.pack()) after ordering, XOR fanins stored positive with
// the parity moved to the result, and the same constant / idempotence /
// complement folding -- so circuits built here are gate-for-gate the
// reference's (sub-miter extraction, AIGER ingest, XOR recovery).
#pragma once

#include <cstdint>
#include <unordered_map>
#include <vector>

namespace es {

struct Lit {
    int32_t node;
    bool neg;
    uint32_t pack() const { return (uint32_t)node * 2u + (neg ? 1u : 0u); }
    bool operator==(const Lit &o) const { return node == o.node && neg == o.neg; }
};

constexpr Lit kFalse{0, false};
constexpr Lit kTrue{0, true};

struct Builder {  // XagBuilder (xag.py:128-192)
    int num_pis;
    std::vector<uint8_t> kind;
    std::vector<uint32_t> in0, in1;
    std::unordered_map<uint64_t, int32_t> table;
    explicit Builder(int n) : num_pis(n) {}
    int32_t num_nodes() const { return 1 + num_pis + (int32_t)kind.size(); }
    Lit node(int k, Lit a, Lit b) {
        Lit lo = a, hi = b;
        if (b.pack() < a.pack()) { lo = b; hi = a; }
        const uint64_t key = ((uint64_t)k << 62) | ((uint64_t)lo.pack() << 31) | hi.pack();
        auto it = table.find(key);
        if (it != table.end()) return Lit{it->second, false};
        const int32_t v = num_nodes();
        kind.push_back((uint8_t)k);
        in0.push_back(lo.pack());
        in1.push_back(hi.pack());
        table.emplace(key, v);
        return Lit{v, false};
    }
    Lit add_and(Lit a, Lit b) {
        if (a == kFalse || b == kFalse) return kFalse;
        if (a == kTrue) return b;
        if (b == kTrue) return a;
        if (a == b) return a;
        if (a.node == b.node) return kFalse;
        return node(0, a, b);
    }
    Lit add_xor(Lit a, Lit b) {
        if (a.node == 0) return a.neg ? Lit{b.node, !b.neg} : b;
        if (b.node == 0) return b.neg ? Lit{a.node, !a.neg} : a;
        if (a == b) return kFalse;
        if (a.node == b.node) return kTrue;
        Lit l = node(1, Lit{a.node, false}, Lit{b.node, false});
        return Lit{l.node, a.neg != b.neg};
    }
};


// A whole XAG: packed literals node*2+neg, kind 0 AND / 1 XOR, outputs.
struct XagC {
    int32_t num_pis = 0;
    std::vector<uint8_t> kind;
    std::vector<uint32_t> in0, in1;
    std::vector<uint32_t> outs;
};

}  // namespace es
