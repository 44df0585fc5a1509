// es_codegen_t.h -- K1T code generation (internal).
#pragma once

#include <string>
#include <vector>

#include "es_core.h"

namespace es {

// Default iterations per phase-1 block (k1t_skeleton.cu ES_TB).
constexpr int kK1TBlock = 16;

struct TSplit {
    std::vector<int> lut_idx;   // node -> LUT index or -1
    std::vector<uint8_t> uni;   // node is word-uniform
    std::vector<int> bidx;      // node -> boundary slot or -1
    std::vector<int> boundary;  // boundary nodes in slot order
    int n_uniform = 0;          // word-uniform LUTs
};

TSplit split_uniform(const LutNet &net);
std::string emit_body_t1(const LutNet &net, const TSplit &t, const std::string &wbq_lo,
                         const std::string &wbq_hi, const std::string &s_store, int tb);
std::string emit_body_t2(const LutNet &net, const TSplit &t, const std::string &out,
                         const std::string &wb_lo, const std::string &wb_hi, const std::string &lane,
                         const std::string &pow2, const std::string &one, const std::string &s_q,
                         int tb);

}  // namespace es
