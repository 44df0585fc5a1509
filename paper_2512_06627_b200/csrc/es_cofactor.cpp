// es_cofactor.cpp -- cofactor expansion of the miter for K1.
//
// The reference evaluates every gate once per 64-pattern word
// (es.py:175-229); K1 evaluates one LUT per 32-pattern word.  Inside a word
// only PIs 1..5 vary; a PI >= 6 is one value for the whole word.  Pick k such
// PIs and let one kernel iteration evaluate the 2^k words that differ only in
// them: within copy c those PIs are constants, so every gate in their
// transitive fanout folds (a partial product b15 & a_i is 0 or a_i), and
// every gate outside it is the same in all copies and is evaluated once.
// Structural hashing across the copies finds the shared logic; constant
// propagation does the folding.  The kernel's word index then enumerates the
// other n-5-k PIs only.
//
// For the 16x16 array-vs-Booth miter, PIs b15, b14, b13 (the multiplier's
// top bits, smallest fanout) give 8 copies for 3,163 LUTs: 395 LUTs per word
// instead of 1,549.
#include <algorithm>
#include <cstdlib>
#include <unordered_map>

#include "es_core.h"

namespace es {

namespace {

// Literal = node*2 + complement; 0 = FALSE, 1 = TRUE.
// Open-addressing (linear probing) structural-hash table: the expansion runs
// for every candidate depth of every config-4 cone (K2's cofactor search), so
// it is a host hot spot (std::unordered_map measured ~5x slower).
struct Strash {
    Dag *d;
    std::vector<uint64_t> keys;  // 0 = empty (a real key always has b >= 2)
    std::vector<int32_t> vals;
    size_t used = 0, mask = 0;
    explicit Strash(Dag *dag) : d(dag) {}
    void reserve(size_t n) {
        size_t cap = 64;
        while (cap < 2 * n) cap <<= 1;
        keys.assign(cap, 0);
        vals.assign(cap, 0);
        mask = cap - 1;
        used = 0;
    }
    static size_t hash(uint64_t k) {
        k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33;
        return (size_t)k;
    }
    void grow() {
        std::vector<uint64_t> ok;
        std::vector<int32_t> ov;
        ok.swap(keys);
        ov.swap(vals);
        keys.assign(ok.size() * 2, 0);
        vals.assign(ok.size() * 2, 0);
        mask = keys.size() - 1;
        for (size_t i = 0; i < ok.size(); ++i) {
            if (!ok[i]) continue;
            size_t h = hash(ok[i]) & mask;
            while (keys[h]) h = (h + 1) & mask;
            keys[h] = ok[i];
            vals[h] = ov[i];
        }
    }
    int32_t node(bool x, uint32_t a, uint32_t b) {
        const uint64_t key = ((uint64_t)x << 63) | ((uint64_t)a << 32) | b;
        if (keys.empty()) reserve(1024);
        size_t h = hash(key) & mask;
        while (keys[h]) {
            if (keys[h] == key) return vals[h];
            h = (h + 1) & mask;
        }
        const int32_t v = d->num_nodes();
        d->is_xor.push_back(x);
        d->f0.push_back((int32_t)(a >> 1));
        d->n0.push_back(a & 1);
        d->f1.push_back((int32_t)(b >> 1));
        d->n1.push_back(b & 1);
        keys[h] = key;
        vals[h] = v;
        if (++used * 2 > keys.size()) grow();
        return v;
    }
    uint32_t mk_and(uint32_t a, uint32_t b) {
        if (a == 0 || b == 0) return 0;
        if (a == 1) return b;
        if (b == 1) return a;
        if (a == b) return a;
        if ((a ^ b) == 1) return 0;
        if (a > b) std::swap(a, b);
        return (uint32_t)node(false, a, b) * 2;
    }
    uint32_t mk_xor(uint32_t a, uint32_t b) {
        if (a <= 1) return b ^ a;
        if (b <= 1) return a ^ b;
        if (a == b) return 0;
        if ((a ^ b) == 1) return 1;
        const uint32_t par = (a ^ b) & 1;
        a &= ~1u;
        b &= ~1u;
        if (a > b) std::swap(a, b);
        return (uint32_t)node(true, a, b) * 2 | par;
    }
};

std::vector<uint8_t> output_cone(const Dag &dag) {
    const int N = dag.num_nodes(), FG = dag.first_gate();
    std::vector<uint8_t> cone(N, 0);
    if (dag.outs.empty()) cone[dag.out_node] = 1;
    for (int32_t o : dag.outs) cone[o] = 1;
    for (int v = N - 1; v >= FG; --v) {
        if (!cone[v]) continue;
        cone[dag.f0[v - FG]] = cone[dag.f1[v - FG]] = 1;
    }
    return cone;
}

}  // namespace

std::vector<int32_t> rank_cofactor_pis(const Dag &dag, int k, int max_pi) {
    // cost of cofactoring PI j ~ the gates whose support contains j (they are
    // duplicated per copy; the rest is shared); PIs <= 40 fit one 64-bit mask
    const int N = dag.num_nodes(), FG = dag.first_gate(), P = dag.num_pis;
    const std::vector<uint8_t> cone = output_cone(dag);
    std::vector<uint64_t> sup(N, 0);
    for (int j = 1; j <= P; ++j) sup[j] = 1ull << j;
    std::vector<int64_t> tfo(P + 1, 0);
    for (int v = FG; v < N; ++v) {
        if (!cone[v]) continue;
        const uint64_t m = sup[dag.f0[v - FG]] | sup[dag.f1[v - FG]];
        sup[v] = m;
        for (uint64_t r = m; r; r &= r - 1) tfo[__builtin_ctzll(r)]++;
    }
    std::vector<int32_t> cand;
    for (int j = kLanePis + 1; j <= std::min(P, max_pi); ++j)
        if (cone[j]) cand.push_back(j);
    std::stable_sort(cand.begin(), cand.end(), [&](int32_t a, int32_t b) {
        if (tfo[a] != tfo[b]) return tfo[a] < tfo[b];
        return a > b;  // ties: the higher PI (later in the pattern order)
    });
    if ((int)cand.size() > k) cand.resize(k);
    if (const char *e = getenv("ES_COF_PIS")) {  // experiment: explicit cofactor PIs
        std::vector<int32_t> forced;
        for (const char *q = e; *q;) {
            forced.push_back(atoi(q));
            while (*q && *q != ',') ++q;
            if (*q == ',') ++q;
        }
        bool below = true;
        for (int32_t j : forced) below = below && j <= max_pi;
        if ((int)forced.size() >= k && below) { forced.resize(k); return forced; }
    }
    return cand;
}

void cofactor_expand(const Dag &dag, const std::vector<int32_t> &pis, Dag *out,
                     const std::vector<int32_t> *copies) {
    const int N = dag.num_nodes(), FG = dag.first_gate(), P = dag.num_pis;
    const std::vector<uint8_t> cone = output_cone(dag);
    *out = Dag();
    out->num_pis = P;
    Strash sh(out);
    sh.reserve((size_t)N * 2);
    const int k = (int)pis.size();
    // gates in the transitive fanout of the cofactor PIs: the only ones that
    // differ between copies; the rest keep copy 0's literal
    std::vector<uint8_t> tfo(N, 0);
    for (int32_t j : pis) tfo[j] = 1;
    std::vector<int32_t> tgates, all;
    for (int v = FG; v < N; ++v) {
        if (!cone[v]) continue;
        all.push_back(v);
        const int g = v - FG;
        if (tfo[dag.f0[g]] || tfo[dag.f1[g]]) { tfo[v] = 1; tgates.push_back(v); }
    }
    std::vector<uint32_t> lit(N, 0);
    std::vector<int32_t> src_outs = dag.outs;
    std::vector<uint8_t> src_neg = dag.outs_neg;
    if (src_outs.empty()) { src_outs.push_back(dag.out_node); src_neg.push_back(dag.out_neg); }
    for (int j = 1; j <= P; ++j) lit[j] = (uint32_t)j * 2;
    std::vector<int32_t> every;
    if (!copies) {
        for (int c = 0; c < (1 << k); ++c) every.push_back(c);
        copies = &every;
    }
    bool first = true;
    for (int32_t c : *copies) {
        for (int b = 0; b < k; ++b) lit[pis[b]] = (uint32_t)((c >> b) & 1);
        // the first copy builds the logic outside the cofactor PIs' fanout too
        for (int v : (first ? all : tgates)) {
            const int g = v - FG;
            const uint32_t a = lit[dag.f0[g]] ^ dag.n0[g], b = lit[dag.f1[g]] ^ dag.n1[g];
            lit[v] = dag.is_xor[g] ? sh.mk_xor(a, b) : sh.mk_and(a, b);
        }
        first = false;
        for (size_t q = 0; q < src_outs.size(); ++q) {
            const uint32_t o = lit[src_outs[q]] ^ src_neg[q];
            out->outs.push_back((int32_t)(o >> 1));
            out->outs_neg.push_back(o & 1);
        }
    }
    out->out_node = out->outs[0];
    out->out_neg = out->outs_neg[0];
}

void map_cofactored(const Dag &dag, const std::vector<int32_t> &pis, LutNet *net,
                    const std::vector<int32_t> *copies) {
    if (pis.empty()) { map_luts(dag, net); return; }
    Dag x;
    cofactor_expand(dag, pis, &x, copies);
    map_luts(x, net);
    net->cof_pis = pis;
    if (copies && (int)copies->size() != (1 << pis.size())) net->copy_ids = *copies;
    const int P = dag.num_pis;
    net->pi_bit.assign(P + 1, -1);
    int bit = 0;
    for (int j = kLanePis + 1; j <= P; ++j) {
        if (std::find(pis.begin(), pis.end(), j) != pis.end()) continue;
        net->pi_bit[j] = (int8_t)bit++;
    }
}

}  // namespace es
