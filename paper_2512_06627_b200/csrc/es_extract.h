// es_extract.h -- sub-miter extraction (internal).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "es_core.h"
#include "es_k2prog.h"

namespace es {

// One extracted and compiled sub-miter.
struct SubMiterC {
    int32_t num_pis = 0;
    std::vector<uint8_t> kind;
    std::vector<uint32_t> in0, in1;
    uint32_t out_lit = 0;
    std::vector<int32_t> pi_map;  // sub PI i+1 -> parent PI pi_map[i]
    uint64_t hash = 0;            // structural hash of the sub-XAG
    bool too_many_inputs = false;
    // reference program (es.py:87-163)
    std::vector<int8_t> op;
    std::vector<int32_t> dst, src0, src1, pi;
    std::vector<uint8_t> neg0, neg1;
    int32_t num_registers = 0;
    int32_t G = 0;  // AND + XOR instructions (the credited gate count)
    K2Prog k2;  // interpreter program (with cofactor copies), built by prepare_k2
    bool k2_ready = false;
    es_prog view() const;
};

int extract_compile(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, int32_t n_merges, const int32_t *merge_node,
                    const uint32_t *merge_lit, int32_t n_pairs, const int32_t *a,
                    const int32_t *b, const uint8_t *polarity, int32_t n_threads,
                    std::vector<SubMiterC> *out, std::string *err);

int evaluate_sub(const SubMiterC &s, uint64_t pattern);
// Build the K2 programs of the sub-miters that lack one, on n_threads host
// threads (0 = all).  Done once per batch, after any selection.
// search = false: plain programs (no cofactor-depth search) -- cheaper on the
// host when the batch's device work is small (a sweep round).
int prepare_k2(std::vector<SubMiterC> &subs, int n_threads, const std::vector<int> *only = nullptr,
               bool search = true);

}  // namespace es
