// es_extract.cpp -- sub-miter extraction + compilation in C++ (SURVEY 8(f)
// next-2): the sweep's per-pair host work, multi-threaded.
//
//  extract : cecprove/sweep.py:92-158 (extract_submiter), step for step --
//            merge resolution (:84-89), support scan (:104-118), dense PI
//            renumbering (:120-121), iterative post-order rebuild of both
//            cones through a structurally hashed builder (:133-152), the
//            pair XOR and polarity (:154-158).
//  builder : cecprove/xag.py:128-192 (XagBuilder) -- same strash key and
//            local rewrites, so sub-miters are gate-for-gate the reference's.
//  compile : es_compile.cpp:ref_compile (es.py:87-163).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "es_core.h"
#include "es_extract.h"
#include "es_xag.h"

namespace es {

namespace {

struct Parent {
    int num_pis;
    int num_gates;
    const uint8_t *kind;
    const uint32_t *in0, *in1;
    std::unordered_map<int32_t, Lit> merges;
    int first() const { return 1 + num_pis; }
    bool is_pi(int v) const { return v >= 1 && v <= num_pis; }
};

std::pair<int32_t, bool> resolve(const Parent &P, int32_t node) {  // sweep.py:84-89
    bool neg = false;
    for (size_t hops = 0;; ++hops) {
        if (hops > P.merges.size()) throw std::runtime_error("cyclic merge map");
        auto it = P.merges.find(node);
        if (it == P.merges.end()) return {node, neg};
        node = it->second.node;
        neg = neg != it->second.neg;
    }
}

uint64_t xag_hash(const SubMiterC &s) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h ^= v; h *= 1099511628211ull; h ^= h >> 29; };
    mix((uint64_t)s.num_pis);
    for (size_t i = 0; i < s.kind.size(); ++i) mix(((uint64_t)s.kind[i] << 62) ^ ((uint64_t)s.in0[i] << 31) ^ s.in1[i]);
    mix(s.out_lit);
    return h;
}

void extract_one(const Parent &P, int32_t a, int32_t b, bool polarity, SubMiterC *out) {
    auto ra = resolve(P, a), rb = resolve(P, b);
    const int32_t an = ra.first, bn = rb.first;
    // support scan (sweep.py:104-118)
    std::vector<int32_t> support;
    std::unordered_set<int32_t> seen;
    std::vector<int32_t> stack{an, bn};
    while (!stack.empty()) {
        const int32_t v = stack.back();
        stack.pop_back();
        if (v == 0 || seen.count(v)) continue;
        seen.insert(v);
        if (P.is_pi(v)) { support.push_back(v); continue; }
        const int g = v - P.first();
        stack.push_back(resolve(P, (int32_t)(P.in0[g] >> 1)).first);
        stack.push_back(resolve(P, (int32_t)(P.in1[g] >> 1)).first);
    }
    std::sort(support.begin(), support.end());
    std::unordered_map<int32_t, int32_t> pi_index;
    for (size_t i = 0; i < support.size(); ++i) pi_index[support[i]] = (int32_t)i + 1;
    Builder bld((int)support.size());
    std::unordered_map<int32_t, Lit> memo;
    memo[0] = kFalse;
    auto mapped = [&](uint32_t packed) {
        auto r = resolve(P, (int32_t)(packed >> 1));
        const Lit got = memo.at(r.first);
        return Lit{got.node, (got.neg != r.second) != (bool)(packed & 1)};
    };
    // iterative post-order rebuild (sweep.py:133-152)
    seen.clear();
    std::vector<std::pair<int32_t, bool>> st{{an, false}, {bn, false}};
    while (!st.empty()) {
        const auto [v, expanded] = st.back();
        st.pop_back();
        if (v == 0 || memo.count(v)) continue;
        if (P.is_pi(v)) { memo[v] = Lit{pi_index[v], false}; continue; }
        const int g = v - P.first();
        if (expanded) {
            const Lit l0 = mapped(P.in0[g]), l1 = mapped(P.in1[g]);
            memo[v] = P.kind[g] == 0 ? bld.add_and(l0, l1) : bld.add_xor(l0, l1);
            continue;
        }
        if (seen.count(v)) continue;
        seen.insert(v);
        st.push_back({v, true});
        st.push_back({resolve(P, (int32_t)(P.in0[g] >> 1)).first, false});
        st.push_back({resolve(P, (int32_t)(P.in1[g] >> 1)).first, false});
    }
    const Lit la{memo[an].node, memo[an].neg != ra.second};
    const Lit lb{memo[bn].node, memo[bn].neg != rb.second};
    Lit o = bld.add_xor(la, lb);
    if (polarity) o.neg = !o.neg;
    out->num_pis = bld.num_pis;
    out->kind = std::move(bld.kind);
    out->in0 = std::move(bld.in0);
    out->in1 = std::move(bld.in1);
    out->out_lit = o.pack();
    out->pi_map = std::move(support);
    out->hash = xag_hash(*out);
}

}  // namespace

int extract_compile(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, int32_t n_merges, const int32_t *merge_node,
                    const uint32_t *merge_lit, int32_t n_pairs, const int32_t *a,
                    const int32_t *b, const uint8_t *polarity, int32_t n_threads,
                    std::vector<SubMiterC> *out, std::string *err) {
    Parent P;
    P.num_pis = num_pis;
    P.num_gates = num_gates;
    P.kind = kind;
    P.in0 = in0;
    P.in1 = in1;
    const int nn = 1 + num_pis + num_gates;
    for (int i = 0; i < n_merges; ++i) P.merges[merge_node[i]] = Lit{(int32_t)(merge_lit[i] >> 1), (bool)(merge_lit[i] & 1)};
    for (int i = 0; i < num_gates; ++i) {
        const int v = 1 + num_pis + i;
        if ((int)(in0[i] >> 1) >= v || (int)(in1[i] >> 1) >= v) { *err = "parent XAG not topological"; return ES_E_BAD_PROGRAM; }
    }
    for (int i = 0; i < n_pairs; ++i)
        if (a[i] < 0 || a[i] >= nn || b[i] < 0 || b[i] >= nn) { *err = "pair node out of range"; return ES_E_BAD_ARG; }
    out->assign(n_pairs, SubMiterC());
    std::atomic<int> next{0};
    std::atomic<int> bad{0};
    auto work = [&]() {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= n_pairs) return;
            SubMiterC &s = (*out)[i];
            try {
                extract_one(P, a[i], b[i], polarity && polarity[i], &s);
            } catch (...) {  // e.g. a merge map that is not a DAG (sweep.py would KeyError)
                bad.fetch_add(1);
                continue;
            }
            if (s.num_pis > ES_MAX_PIS) { s.too_many_inputs = true; continue; }
            const size_t cap = (size_t)s.num_pis + s.kind.size() + 1;
            s.op.resize(cap); s.dst.resize(cap); s.src0.resize(cap); s.neg0.resize(cap);
            s.src1.resize(cap); s.neg1.resize(cap); s.pi.resize(cap);
            const int n = ref_compile(s.num_pis, (int32_t)s.kind.size(), s.kind.data(), s.in0.data(),
                                      s.in1.data(), s.out_lit, s.op.data(), s.dst.data(), s.src0.data(),
                                      s.neg0.data(), s.src1.data(), s.neg1.data(), s.pi.data(),
                                      &s.num_registers);
            if (n < 0) { bad.fetch_add(1); continue; }
            s.op.resize(n); s.dst.resize(n); s.src0.resize(n); s.neg0.resize(n);
            s.src1.resize(n); s.neg1.resize(n); s.pi.resize(n);
            for (int8_t o : s.op) s.G += o == ES_OP_AND || o == ES_OP_XOR;
            Dag dag;
            std::string e2;
            if (build_dag(s.view(), &dag, &e2) != ES_OK) { bad.fetch_add(1); continue; }
        }
    };
    int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = std::min(T, std::max(1, n_pairs / 8));
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    if (bad.load()) { *err = "sub-miter extraction/compile failed (cyclic merges?)"; return ES_E_BAD_PROGRAM; }
    return ES_OK;
}

es_prog SubMiterC::view() const {
    es_prog p;
    p.num_instrs = (int32_t)op.size();
    p.num_registers = num_registers;
    p.num_pis = num_pis;
    p.op = op.data();
    p.dst = dst.data();
    p.src0 = src0.data();
    p.neg0 = neg0.data();
    p.src1 = src1.data();
    p.neg1 = neg1.data();
    p.pi = pi.data();
    return p;
}

int evaluate_sub(const SubMiterC &s, uint64_t pattern) {  // eval.py:22-36 on the witness
    std::vector<uint8_t> v(1 + s.num_pis + s.kind.size(), 0);
    for (int i = 0; i < s.num_pis; ++i) v[1 + i] = (pattern >> i) & 1;
    for (size_t g = 0; g < s.kind.size(); ++g) {
        const int x = v[s.in0[g] >> 1] ^ (s.in0[g] & 1), y = v[s.in1[g] >> 1] ^ (s.in1[g] & 1);
        v[1 + s.num_pis + g] = s.kind[g] == 0 ? (x & y) : (x ^ y);
    }
    return v[s.out_lit >> 1] ^ (s.out_lit & 1);
}

int prepare_k2(std::vector<SubMiterC> &subs, int n_threads, const std::vector<int> *only, bool search) {
    std::vector<int> todo;
    if (only) {
        for (int i : *only)
            if (!subs[i].k2_ready && !subs[i].too_many_inputs) todo.push_back(i);
    } else {
        for (int i = 0; i < (int)subs.size(); ++i)
            if (!subs[i].k2_ready && !subs[i].too_many_inputs) todo.push_back(i);
    }
    if (todo.empty()) return ES_OK;
    std::atomic<int> next{0}, bad{0};
    auto work = [&]() {
        for (;;) {
            const int q = next.fetch_add(1);
            if (q >= (int)todo.size()) return;
            SubMiterC &s = subs[todo[q]];
            Dag dag;
            std::string err;
            if (build_dag(s.view(), &dag, &err) != ES_OK) { bad.fetch_add(1); continue; }
            if (search) build_k2prog_auto(dag, &s.k2);
            else build_k2prog(dag, &s.k2);
            s.k2_ready = true;
        }
    };
    int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = std::min<int>(T, std::max<int>(1, (int)todo.size() / 8));
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    return bad.load() ? ES_E_BAD_PROGRAM : ES_OK;
}

}  // namespace es
