// es_codegen_t.cpp -- PTX bodies of K1T (k1t_skeleton.cu).
//
// Splits the mapped LUT network into
//   * word-uniform LUTs: support avoids PIs 1..5, so every bit of a 32-bit word
//     carries the same value; evaluated in phase 1 as super-words (bit L = lane
//     L's word), once per ES_TB iterations per lane;
//   * per-lane LUTs: everything else, evaluated in phase 2 per iteration.
// Boundary = word-uniform LUTs read by a per-lane LUT (or the output); only
// those cross shared memory.
#include <sstream>
#include <unordered_map>

#include "es_codegen_t.h"

namespace es {

TSplit split_uniform(const LutNet &net) {
    TSplit t;
    const int N = (int)net.is_const.size(), P = net.num_pis;
    t.lut_idx.assign(N, -1);
    for (size_t i = 0; i < net.luts.size(); ++i) t.lut_idx[net.luts[i].node] = (int)i;
    t.uni.assign(N, 0);
    for (int v = 0; v < N; ++v) {
        if (v >= 6 && v <= P) t.uni[v] = 1;  // word PIs
        else if (net.is_const[v] && (net.const_val[v] == 0u || net.const_val[v] == ~0u)) t.uni[v] = 1;
    }
    for (const Lut &L : net.luts) {
        bool u = true;
        for (int q = 0; q < 3; ++q) u = u && t.uni[L.leaf[q]];
        t.uni[L.node] = u;
        t.n_uniform += u;
    }
    t.bidx.assign(N, -1);
    auto mark = [&](int v) {
        if (t.lut_idx[v] >= 0 && t.uni[v] && t.bidx[v] < 0) {
            t.bidx[v] = (int)t.boundary.size();
            t.boundary.push_back(v);
        }
    };
    for (const Lut &L : net.luts)
        if (!t.uni[L.node])
            for (int q = 0; q < 3; ++q) mark(L.leaf[q]);
    mark(net.out_node);
    return t;
}

namespace {

struct Consts {
    std::unordered_map<uint32_t, int> idx;
    std::vector<uint32_t> vals;
    std::string name(const char *prefix, uint32_t c) {
        auto it = idx.find(c);
        int k;
        if (it == idx.end()) { k = (int)vals.size(); idx[c] = k; vals.push_back(c); }
        else k = it->second;
        return std::string(prefix) + std::to_string(k);
    }
};

// uniform masks of word PIs >= 11 from a word-block index (bit j-11)
void emit_block_pis(std::ostringstream &s, const char *reg, const std::vector<uint8_t> &used, int P,
                    const std::string &lo, const std::string &hi) {
    for (int j = 11; j <= P; ++j)
        if (used[j]) {
            const int bit = j - 11;
            s << "shl.b32 " << reg << j << ", " << (bit < 32 ? lo : hi) << ", " << (31 - (bit & 31)) << ";\n";
            s << "shr.s32 " << reg << j << ", " << reg << j << ", 31;\n";
        }
}

}  // namespace

std::string emit_body_t1(const LutNet &net, const TSplit &t, const std::string &wbq_lo,
                         const std::string &wbq_hi, const std::string &s_store, int tb) {
    const int P = net.num_pis;
    Consts K;
    std::vector<uint8_t> pi_used(P + 1, 0);
    auto name = [&](int v) -> std::string {
        if (t.lut_idx[v] >= 0) return "%etq" + std::to_string(t.lut_idx[v]);
        if (v >= 6 && v <= 10 && v <= P) return K.name("%etk", kLaneMask[v - 6]);  // lane patterns
        if (v >= 11 && v <= P) { pi_used[v] = 1; return "%etm" + std::to_string(v); }
        return K.name("%etk", net.const_val[v]);
    };
    std::ostringstream body;
    for (const Lut &L : net.luts) {
        if (!t.uni[L.node]) continue;
        const int i = t.lut_idx[L.node];
        body << "lop3.b32 %etq" << i << ", " << name(L.leaf[2]) << ", " << name(L.leaf[1]) << ", "
             << name(L.leaf[0]) << ", " << (int)L.tt << ";\n";
        if (t.bidx[L.node] >= 0)
            body << "st.shared.u32 [" << s_store << "+" << (t.bidx[L.node] * tb * 4) << "], %etq" << i << ";\n";
    }
    std::ostringstream s;
    s << "{\n";
    if (!net.luts.empty()) s << ".reg .b32 %etq<" << net.luts.size() << ">;\n";
    s << ".reg .b32 %etm<" << (P + 1) << ">;\n";
    std::string b = body.str();
    if (!K.vals.empty()) s << ".reg .b32 %etk<" << K.vals.size() << ">;\n";
    for (size_t k = 0; k < K.vals.size(); ++k) s << "mov.b32 %etk" << k << ", " << K.vals[k] << ";\n";
    emit_block_pis(s, "%etm", pi_used, P, wbq_lo, wbq_hi);
    s << b << "}\n";
    return s.str();
}

std::string emit_body_t2(const LutNet &net, const TSplit &t, const std::string &out,
                         const std::string &wb_lo, const std::string &wb_hi, const std::string &lane,
                         const std::string &pow2, const std::string &one, const std::string &s_q,
                         int tb) {
    const int N = (int)net.is_const.size(), P = net.num_pis;
    Consts K;
    std::vector<uint8_t> pi_used(P + 1, 0), pi_lane(P + 1, 0), loaded(N, 0);
    std::ostringstream body;
    auto name = [&](int v) -> std::string {
        if (t.lut_idx[v] >= 0) {
            const int i = t.lut_idx[v];
            if (!t.uni[v]) return "%esq" + std::to_string(i);
            if (!loaded[v]) {  // boundary super-word: load, move bit L to the sign, spread
                loaded[v] = 1;
                body << "ld.shared.u32 %esx" << i << ", [" << s_q << "+" << (t.bidx[v] * tb * 4) << "];\n"
                     << "mul.lo.u32 %esx" << i << ", %esx" << i << ", " << pow2 << ";\n"
                     << "mul.hi.s32 %esx" << i << ", %esx" << i << ", " << one << ";\n";
            }
            return "%esx" + std::to_string(i);
        }
        if (net.is_const[v]) return K.name("%esk", net.const_val[v]);
        if (v >= 6 && v <= 10) { pi_lane[v] = 1; return "%esl" + std::to_string(v); }
        pi_used[v] = 1;
        return "%esm" + std::to_string(v);
    };
    for (const Lut &L : net.luts) {
        if (t.uni[L.node]) continue;
        const std::string a = name(L.leaf[2]), b = name(L.leaf[1]), c = name(L.leaf[0]);
        body << "lop3.b32 %esq" << t.lut_idx[L.node] << ", " << a << ", " << b << ", " << c << ", "
             << (int)L.tt << ";\n";
    }
    const std::string oname = name(net.out_node);
    std::ostringstream s;
    s << "{\n";
    if (!net.luts.empty()) {
        s << ".reg .b32 %esq<" << net.luts.size() << ">;\n";
        s << ".reg .b32 %esx<" << net.luts.size() << ">;\n";
    }
    s << ".reg .b32 %esm<" << (P + 1) << ">;\n.reg .b32 %esl<" << (P + 1) << ">;\n";
    std::string b = body.str();
    if (!K.vals.empty()) s << ".reg .b32 %esk<" << K.vals.size() << ">;\n";
    for (size_t k = 0; k < K.vals.size(); ++k) s << "mov.b32 %esk" << k << ", " << K.vals[k] << ";\n";
    for (int j = 6; j <= std::min(P, 10); ++j)
        if (pi_lane[j]) {
            s << "shl.b32 %esl" << j << ", " << lane << ", " << (31 - (j - 6)) << ";\n";
            s << "shr.s32 %esl" << j << ", %esl" << j << ", 31;\n";
        }
    emit_block_pis(s, "%esm", pi_used, P, wb_lo, wb_hi);
    s << b;
    if (net.out_neg) s << "not.b32 " << out << ", " << oname << ";\n";
    else s << "mov.b32 " << out << ", " << oname << ";\n";
    s << "}\n";
    return s.str();
}

}  // namespace es
