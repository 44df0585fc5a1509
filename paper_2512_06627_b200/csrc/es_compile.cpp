// es_compile.cpp -- host compiler of the B200 ES engine.
//
//  * ref_compile : compile_program (cecprove/es.py:87-163), instruction-exact:
//                  output-cone marking (:103-111), fanin refcounts (:113-119),
//                  topological emission with lazy PI loads (:138-150), fanins
//                  consumed before dst allocation (:151-156), LIFO pool
//                  (:126-136), output-is-PI (:160-161), constant output (:99-101).
//  * build_dag   : the register program back to an SSA graph, so any
//                  InstrProgram (the reference's seam) can be run.
//  * map_luts    : LUT-3 cover of the cone.  A LOP3 evaluates any 3-input
//                  function of 32-bit words in one ALU issue, so covering the
//                  XAG with 3-feasible cuts cuts the issue count well below the
//                  gate count (a full adder is 2 LOP3 instead of 5 gates).
//                  Low PIs 1..5 are per-bit constants of a 32-bit word
//                  (0xAAAAAAAA ...): nodes over them fold to constants.
//  * schedule    : DFS order that keeps the live set small enough to stay in
//                  registers (the reason the reference recycles registers,
//                  es.py:9-10; here the register file is the SM's).
//  * emit_body_ptx / eval_lutnet : the kernel body and its CPU model.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <sstream>
#include <unordered_map>

#include "es_core.h"

namespace es {

const uint32_t kLaneMask[kLanePis] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u,
                                      0xFF00FF00u, 0xFFFF0000u};

uint32_t lane_valid_mask(int num_pis) {
    return num_pis >= kLanePis ? 0xFFFFFFFFu : ((1u << (1u << num_pis)) - 1u);
}

// ---------------------------------------------------------------------------
// compile_program, reference schedule (es.py:87-163)
// ---------------------------------------------------------------------------
int32_t ref_compile(int32_t num_pis, int32_t num_gates, const uint8_t *kind,
                    const uint32_t *in0, const uint32_t *in1, uint32_t out_lit,
                    int8_t *op, int32_t *dst, int32_t *src0, uint8_t *neg0,
                    int32_t *src1, uint8_t *neg1, int32_t *pi, int32_t *num_registers) {
    if (num_pis > ES_MAX_PIS) return ES_E_TOO_MANY_INPUTS;
    if (num_pis < 0 || num_gates < 0) return ES_E_BAD_PROGRAM;
    const int first = 1 + num_pis, nn = first + num_gates;
    const int onode = (int)(out_lit >> 1);
    const bool oneg = out_lit & 1;
    if (onode >= nn) return ES_E_BAD_PROGRAM;
    int n = 0;
    auto put = [&](int o, int d, int a, bool na, int b, bool nb, int p) {
        op[n] = (int8_t)o; dst[n] = d; src0[n] = a; neg0[n] = na; src1[n] = b;
        neg1[n] = nb; pi[n] = p; ++n;
    };
    if (onode == 0) {
        put(ES_OP_OUTPUT, 0, -1, oneg, -1, false, 0);
        *num_registers = 0;
        return n;
    }
    std::vector<uint8_t> live(nn, 0);
    live[onode] = 1;
    for (int v = nn - 1; v >= first; --v) {
        if (!live[v]) continue;
        const int g = v - first;
        const int a = (int)(in0[g] >> 1), b = (int)(in1[g] >> 1);
        if (a >= v || b >= v || a == 0 || b == 0) return ES_E_BAD_PROGRAM;
        live[a] = live[b] = 1;
    }
    std::vector<int32_t> refs(nn, 0), reg(nn, -1), pool;
    refs[onode] += 1;
    for (int v = first; v < nn; ++v)
        if (live[v]) { refs[in0[v - first] >> 1]++; refs[in1[v - first] >> 1]++; }
    int peak = 0;
    auto alloc = [&]() -> int {
        if (!pool.empty()) { int r = pool.back(); pool.pop_back(); return r; }
        return peak++;
    };
    auto load_pi = [&](int v) {
        if (reg[v] < 0) { reg[v] = alloc(); put(ES_OP_LOAD_PI, reg[v], -1, false, -1, false, v); }
    };
    auto consume = [&](int v) { if (--refs[v] == 0) pool.push_back(reg[v]); };
    for (int v = first; v < nn; ++v) {
        if (!live[v]) continue;
        const int g = v - first;
        const int a = (int)(in0[g] >> 1), b = (int)(in1[g] >> 1);
        if (a <= num_pis) load_pi(a);
        if (b <= num_pis) load_pi(b);
        const int ra = reg[a], rb = reg[b];
        consume(a);
        consume(b);
        reg[v] = alloc();
        put(kind[g] ? ES_OP_XOR : ES_OP_AND, reg[v], ra, in0[g] & 1, rb, in1[g] & 1, 0);
    }
    if (onode <= num_pis) load_pi(onode);
    put(ES_OP_OUTPUT, 0, reg[onode], oneg, -1, false, 0);
    *num_registers = peak;
    return n;
}

// ---------------------------------------------------------------------------
// register program -> SSA graph
// ---------------------------------------------------------------------------
int build_dag(const es_prog &p, Dag *dag, std::string *err) {
    auto fail = [&](const std::string &m) { if (err) *err = m; return ES_E_BAD_PROGRAM; };
    if (p.num_pis < 0) return fail("negative PI count");
    if (p.num_pis > ES_MAX_PIS) return ES_E_TOO_MANY_INPUTS;
    if (p.num_instrs < 1) return fail("empty program");
    if (p.op[p.num_instrs - 1] != ES_OP_OUTPUT) return fail("last instruction is not OUTPUT");
    dag->num_pis = p.num_pis;
    dag->is_xor.clear(); dag->f0.clear(); dag->f1.clear(); dag->n0.clear(); dag->n1.clear();
    const int R = std::max(p.num_registers, 0);
    std::vector<int32_t> node_of(R, -1);
    int next = 1 + p.num_pis;
    for (int i = 0; i < p.num_instrs; ++i) {
        const int o = p.op[i];
        if (o == ES_OP_OUTPUT) {
            if (i != p.num_instrs - 1) return fail("OUTPUT before the end");
            if (p.src0[i] < 0) { dag->out_node = 0; dag->out_neg = p.neg0[i]; break; }
            if (p.src0[i] >= R || node_of[p.src0[i]] < 0) return fail("OUTPUT reads an undefined register");
            dag->out_node = node_of[p.src0[i]];
            dag->out_neg = p.neg0[i];
            break;
        }
        if (p.dst[i] < 0 || p.dst[i] >= R) return fail("dst register out of range");
        if (o == ES_OP_LOAD_PI) {
            if (p.pi[i] < 1 || p.pi[i] > p.num_pis) return fail("LOAD_PI index out of range");
            node_of[p.dst[i]] = p.pi[i];
        } else if (o == ES_OP_AND || o == ES_OP_XOR) {
            const int a = p.src0[i], b = p.src1[i];
            if (a < 0 || a >= R || b < 0 || b >= R || node_of[a] < 0 || node_of[b] < 0)
                return fail("gate reads an undefined register");
            dag->is_xor.push_back(o == ES_OP_XOR);
            dag->f0.push_back(node_of[a]);
            dag->n0.push_back(p.neg0[i] ? 1 : 0);
            dag->f1.push_back(node_of[b]);
            dag->n1.push_back(p.neg1[i] ? 1 : 0);
            node_of[p.dst[i]] = next++;
        } else {
            return fail("unknown opcode");
        }
    }
    return ES_OK;
}

// ---------------------------------------------------------------------------
// LUT-3 mapping
// ---------------------------------------------------------------------------
namespace {

struct Cut {
    int32_t leaf[3];
    uint8_t n;
    uint8_t tt;  // over leaf k = bit k of the minterm index; replicated over unused vars
    float af;
};

inline uint8_t expand_tt(const Cut &c, const int32_t *L, int nL) {
    int pos[3] = {0, 0, 0};
    for (int k = 0; k < c.n; ++k)
        for (int q = 0; q < nL; ++q)
            if (L[q] == c.leaf[k]) pos[k] = q;
    uint8_t r = 0;
    for (int i = 0; i < 8; ++i) {
        int j = 0;
        for (int k = 0; k < c.n; ++k) j |= ((i >> pos[k]) & 1) << k;
        r |= ((c.tt >> j) & 1) << i;
    }
    return r;
}

inline bool depends(uint8_t tt, int k) {
    for (int i = 0; i < 8; ++i)
        if (((tt >> i) & 1) != ((tt >> (i ^ (1 << k))) & 1)) return true;
    return false;
}

inline uint8_t drop_var(uint8_t tt, int k) {
    uint8_t r = 0;
    for (int i = 0; i < 8; ++i) {
        int lo = i & ((1 << k) - 1);
        int src = lo | ((i >> k) << (k + 1));
        src &= 7;
        r |= ((tt >> src) & 1) << i;
    }
    return r;
}

// canonical replicated form of a tt over n vars
inline uint8_t replicate(uint8_t tt, int n) {
    uint8_t r = 0;
    for (int i = 0; i < 8; ++i) r |= ((tt >> (i & ((1 << n) - 1))) & 1) << i;
    return r;
}

inline uint32_t lut3(uint8_t tt, uint32_t a /*leaf2*/, uint32_t b /*leaf1*/, uint32_t c /*leaf0*/) {
    uint32_t r = 0;
    for (int i = 0; i < 8; ++i)
        if ((tt >> i) & 1) r |= ((i & 4) ? a : ~a) & ((i & 2) ? b : ~b) & ((i & 1) ? c : ~c);
    return r;
}

constexpr int kMaxCuts = 10;

}  // namespace

void map_luts(const Dag &dag, LutNet *net) {
    const int N = dag.num_nodes(), FG = dag.first_gate();
    const int P = dag.num_pis;
    net->num_pis = P;
    net->luts.clear();
    net->pis_used.clear();
    net->is_const.assign(N, 0);
    net->const_val.assign(N, 0);
    net->num_gates = 0;
    net->peak_live = 0;
    net->cof_pis.clear();
    net->pi_bit.assign(P + 1, -1);
    for (int j = kLanePis + 1; j <= P; ++j) net->pi_bit[j] = (int8_t)(j - kLanePis - 1);
    std::vector<int32_t> outs = dag.outs;
    std::vector<uint8_t> outs_neg = dag.outs_neg;
    if (outs.empty()) { outs.push_back(dag.out_node); outs_neg.push_back(dag.out_neg); }

    std::vector<uint8_t> cone(N, 0);
    for (int32_t o : outs) cone[o] = 1;
    for (int v = N - 1; v >= FG; --v) {
        if (!cone[v]) continue;
        const int g = v - FG;
        cone[dag.f0[g]] = cone[dag.f1[g]] = 1;
    }
    // constant folding: node 0, lane PIs 1..5, and gates over constants only
    std::vector<uint8_t> &isc = net->is_const;
    std::vector<uint32_t> &cv = net->const_val;
    isc[0] = 1; cv[0] = 0;
    for (int j = 1; j <= std::min(P, kLanePis); ++j) { isc[j] = 1; cv[j] = kLaneMask[j - 1]; }
    std::vector<int32_t> fo(N, 0);
    for (int32_t o : outs) fo[o] += 1;
    for (int v = FG; v < N; ++v) {
        if (!cone[v]) continue;
        const int g = v - FG;
        net->num_gates++;
        fo[dag.f0[g]]++; fo[dag.f1[g]]++;
        const int a = dag.f0[g], b = dag.f1[g];
        if (isc[a] && isc[b]) {
            uint32_t x = cv[a] ^ (dag.n0[g] ? ~0u : 0u), y = cv[b] ^ (dag.n1[g] ? ~0u : 0u);
            isc[v] = 1;
            cv[v] = dag.is_xor[g] ? (x ^ y) : (x & y);
        }
    }
    auto is_gate_lut = [&](int v) { return v >= FG && cone[v] && !isc[v]; };

    // priority cut enumeration in topological order
    std::vector<std::vector<Cut>> cuts(N);
    std::vector<float> af(N, 0.f);
    auto trivial = [](int v) { Cut c{}; c.leaf[0] = v; c.leaf[1] = c.leaf[2] = -1; c.n = 1; c.tt = 0xAA; c.af = 0; return c; };
    for (int v = 1; v <= P; ++v) cuts[v].push_back(trivial(v));
    std::vector<Cut> cand;
    for (int v = FG; v < N; ++v) {
        if (!cone[v]) continue;
        if (isc[v]) { cuts[v].push_back(trivial(v)); continue; }
        const int g = v - FG;
        const int a = dag.f0[g], b = dag.f1[g];
        const bool x = dag.is_xor[g];
        cand.clear();
        const std::vector<Cut> &ca = cuts[a], &cb = cuts[b];
        for (const Cut &c0 : ca) {
            for (const Cut &c1 : cb) {
                int32_t L[3];
                int nL = 0, i = 0, j = 0;
                bool ok = true;
                while (i < c0.n || j < c1.n) {
                    int32_t pick;
                    if (j >= c1.n || (i < c0.n && c0.leaf[i] < c1.leaf[j])) pick = c0.leaf[i++];
                    else if (i >= c0.n || c1.leaf[j] < c0.leaf[i]) pick = c1.leaf[j++];
                    else { pick = c0.leaf[i]; ++i; ++j; }
                    if (nL == 3) { ok = false; break; }
                    L[nL++] = pick;
                }
                if (!ok) continue;
                uint8_t t0 = expand_tt(c0, L, nL), t1 = expand_tt(c1, L, nL);
                if (dag.n0[g]) t0 = ~t0;
                if (dag.n1[g]) t1 = ~t1;
                uint8_t tt = x ? (uint8_t)(t0 ^ t1) : (uint8_t)(t0 & t1);
                // support reduction
                for (int k = nL - 1; k >= 0; --k) {
                    if (!depends(tt, k)) {
                        tt = drop_var(tt, k);
                        for (int q = k; q + 1 < nL; ++q) L[q] = L[q + 1];
                        --nL;
                    }
                }
                Cut c{};
                c.n = (uint8_t)nL;
                for (int q = 0; q < 3; ++q) c.leaf[q] = q < nL ? L[q] : -1;
                c.tt = replicate(tt, nL);
                float s = 1.f;
                for (int q = 0; q < nL; ++q) s += af[L[q]] / (float)std::max(1, fo[L[q]]);
                c.af = s;
                cand.push_back(c);
            }
        }
        // a constant function makes the node a constant
        bool became_const = false;
        for (const Cut &c : cand) {
            if (c.n == 0) {
                isc[v] = 1;
                cv[v] = (c.tt & 1) ? ~0u : 0u;
                became_const = true;
                break;
            }
        }
        if (became_const) { cuts[v].push_back(trivial(v)); continue; }
        std::sort(cand.begin(), cand.end(), [](const Cut &p, const Cut &q) {
            if (p.af != q.af) return p.af < q.af;
            return p.n < q.n;
        });
        std::vector<Cut> &cs = cuts[v];
        for (const Cut &c : cand) {
            bool dup = false;
            for (const Cut &d : cs)
                if (d.n == c.n && d.leaf[0] == c.leaf[0] && d.leaf[1] == c.leaf[1] && d.leaf[2] == c.leaf[2]) { dup = true; break; }
            if (dup) continue;
            cs.push_back(c);
            if ((int)cs.size() >= kMaxCuts) break;
        }
        af[v] = cs.empty() ? 1.f : cs[0].af;
        cs.push_back(trivial(v));  // last: used only as a leaf of fanout cuts
    }

    // cover: best cut per node, then exact-area recovery
    std::vector<int> best(N, 0), mref(N, 0);
    // word-uniform nodes (support avoids the lane PIs): a 2-input LUT over
    // one of them is an FMA-pipe IMAD in emit_body_ptx, so it costs the ALU
    // pipe nothing; `imad_cost` weighs it in the area recovery
    std::vector<uint8_t> uni(N, 0);
    for (int j = kLanePis + 1; j <= P; ++j) uni[j] = 1;
    for (int v = FG; v < N; ++v) {
        if (!cone[v] || isc[v]) continue;
        const int g = v - FG;
        auto u_of = [&](int a) { return isc[a] ? (cv[a] == 0u || cv[a] == ~0u) : uni[a] != 0; };
        uni[v] = u_of(dag.f0[g]) && u_of(dag.f1[g]);
    }
    static const float imad_cost = getenv("ES_IMAD_COST") ? (float)atof(getenv("ES_IMAD_COST")) : 1.0f;
    auto cut_cost = [&](const Cut &c) -> float {
        if (imad_cost == 1.0f || c.n != 2) return 1.0f;
        const bool s0 = !isc[c.leaf[0]] && uni[c.leaf[0]], s1 = !isc[c.leaf[1]] && uni[c.leaf[1]];
        return (s0 || s1) ? imad_cost : 1.0f;
    };
    std::function<float(int, const Cut &)> ref_cut, deref_cut;
    ref_cut = [&](int v, const Cut &c) {
        float area = cut_cost(c);
        for (int q = 0; q < c.n; ++q) {
            int l = c.leaf[q];
            if (is_gate_lut(l) && mref[l]++ == 0) area += ref_cut(l, cuts[l][best[l]]);
        }
        return area;
    };
    deref_cut = [&](int v, const Cut &c) {
        float area = cut_cost(c);
        for (int q = 0; q < c.n; ++q) {
            int l = c.leaf[q];
            if (is_gate_lut(l) && --mref[l] == 0) area += deref_cut(l, cuts[l][best[l]]);
        }
        return area;
    };
    bool any_gate_out = false;
    for (int32_t o : outs) {
        if (!is_gate_lut(o)) continue;
        any_gate_out = true;
        if (mref[o]++ == 0) ref_cut(o, cuts[o][best[o]]);
    }
    if (any_gate_out) {
        for (int pass = 0; pass < 3; ++pass) {
            for (int v = FG; v < N; ++v) {
                if (!is_gate_lut(v) || mref[v] == 0) continue;
                deref_cut(v, cuts[v][best[v]]);
                int bi = best[v];
                float ba = 1e30f;
                float baf = 1e30f;
                const int nc = (int)cuts[v].size() - 1;  // exclude trivial
                for (int ci = 0; ci < nc; ++ci) {
                    float a = ref_cut(v, cuts[v][ci]);
                    deref_cut(v, cuts[v][ci]);
                    if (a < ba || (a == ba && cuts[v][ci].af < baf)) { ba = a; bi = ci; baf = cuts[v][ci].af; }
                }
                best[v] = bi;
                ref_cut(v, cuts[v][best[v]]);
            }
        }
    }

    // schedule: DFS post-order, children by decreasing register need
    std::vector<int> need(N, 0), users(N, 0);
    std::vector<uint8_t> pi_used(P + 1, 0);
    for (int v = FG; v < N; ++v) {
        if (!is_gate_lut(v) || mref[v] == 0) continue;
        const Cut &c = cuts[v][best[v]];
        for (int q = 0; q < c.n; ++q) {
            int l = c.leaf[q];
            if (is_gate_lut(l)) users[l]++;
            else if (l >= 1 && l <= P && !isc[l]) pi_used[l] = 1;
        }
    }
    for (int32_t o : outs)
        if (o >= 1 && o <= P && !isc[o]) pi_used[o] = 1;
    for (int j = 1; j <= P; ++j) if (pi_used[j]) net->pis_used.push_back(j);
    std::vector<int> order;
    if (any_gate_out) {
        // need() bottom-up in topological order
        for (int v = FG; v < N; ++v) {
            if (!is_gate_lut(v) || mref[v] == 0) continue;
            const Cut &c = cuts[v][best[v]];
            int kn[3], k = 0;
            for (int q = 0; q < c.n; ++q) if (is_gate_lut(c.leaf[q])) kn[k++] = need[c.leaf[q]];
            std::sort(kn, kn + k, std::greater<int>());
            int nd = 1;
            for (int q = 0; q < k; ++q) nd = std::max(nd, kn[q] + q);
            need[v] = nd;
        }
    }
    // iterative DFS from each output in turn, highest-need pending child first
    auto dfs = [&](const std::vector<int32_t> &roots) {
        std::vector<uint8_t> dn(N, 0);
        std::vector<int> ord, st;
        for (int32_t o : roots) {
            if (!is_gate_lut(o) || dn[o]) continue;
            st.push_back(o);
            while (!st.empty()) {
                const int v = st.back();
                if (dn[v]) { st.pop_back(); continue; }
                const Cut &c = cuts[v][best[v]];
                int pick = -1;
                for (int q = 0; q < c.n; ++q) {
                    int l = c.leaf[q];
                    if (is_gate_lut(l) && !dn[l] && (pick < 0 || need[l] > need[pick])) pick = l;
                }
                if (pick >= 0) { st.push_back(pick); continue; }
                dn[v] = 1;
                ord.push_back(v);
                st.pop_back();
            }
        }
        return ord;
    };
    // peak simultaneously-live LUT values of an order
    auto peak_of = [&](const std::vector<int> &ord) {
        std::vector<int> rem = users;
        for (int32_t o : outs)
            if (is_gate_lut(o)) rem[o] += 1;
        int live = 0, peak = 0;
        for (int v : ord) {
            const Cut &c = cuts[v][best[v]];
            int freed = 0;
            for (int q = 0; q < c.n; ++q) {
                int l = c.leaf[q];
                bool seen = false;
                for (int r = 0; r < q; ++r) seen |= c.leaf[r] == l;
                if (seen || !is_gate_lut(l)) continue;
                if (--rem[l] == 0) ++freed;
            }
            live = live - freed + 1;
            peak = std::max(peak, live);
        }
        return peak;
    };
    if (any_gate_out) {
        order = dfs(outs);
        if (outs.size() > 1) {
            // cofactor copies: also try the most demanding copies first and keep
            // the order with the smaller live set (fewer spills at 255 registers)
            std::vector<int32_t> by_need = outs;
            std::stable_sort(by_need.begin(), by_need.end(), [&](int a, int b) {
                const int na = is_gate_lut(a) ? need[a] : 0, nb = is_gate_lut(b) ? need[b] : 0;
                return na > nb;
            });
            std::vector<int> alt = dfs(by_need);
            if (peak_of(alt) < peak_of(order)) order.swap(alt);
            // visit the copies in bit-reversed order: logic shared by the copies
            // that agree on a cofactor PI is then used by consecutive copies
            // and dies early (mult16, k=4: peak live 358 -> 212 values, kernel
            // 2.58 -> 2.32 ms, JIT 1.03 -> 0.74 s).  The OUT fold still runs in
            // copy order (flush_outputs waits for copy 0).
            // (a restricted variant's copies 0..C-1 with C not a power of two:
            // the bit-reversed order of the enclosing power of two, truncated)
            const int C = (int)outs.size();
            int kb = 0;
            while ((1 << kb) < C) ++kb;
            // Generalised: the copies are visited as the leaves of a binary
            // tree that splits on the cofactor PIs in some order (bit-reversed
            // = split on PI 0 first).  Logic depending on a set S of cofactor
            // PIs stays live while the copies matching S's values are visited,
            // so the split order decides the live set; try every order of up
            // to 4 PIs (24) and keep the smallest peak.  (5 PIs, 120 orders:
            // mult16 k=5 446 -> 322 live values, but a k=5 body is ~150 KB of
            // SASS and instruction-fetch bound -- ncu stall no_instruction
            // 2.98 per issue, 4.5 ms vs 2.35 at k=4 -- so not worth the
            // mapping time.)
            std::vector<int> perm(kb);
            for (int b = 0; b < kb; ++b) perm[b] = b;
            int best_peak = peak_of(order);
            do {
                std::vector<int32_t> seq;
                for (int c = 0; c < (1 << kb); ++c) {
                    // the c-th leaf: bit t of c (MSB first) is the value of PI perm[t]
                    int r = 0;
                    for (int t = 0; t < kb; ++t) r |= ((c >> (kb - 1 - t)) & 1) << perm[t];
                    if (r < C) seq.push_back(outs[r]);
                }
                std::vector<int> o2 = dfs(seq);
                const int pk = peak_of(o2);
                if (pk < best_peak) { best_peak = pk; order.swap(o2); }
            } while (kb <= 4 && std::next_permutation(perm.begin(), perm.end()));
        }
        if (getenv("ES_LIST_SCHED")) {
            // experiment: greedy list scheduling, prefer the ready node that frees most
            std::vector<int> pos(N, -1);
            for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = (int)i;
            std::vector<int> pend(N, 0), rem = users;
            for (int32_t o : outs) if (is_gate_lut(o)) rem[o] += 1;
            std::vector<std::vector<int>> parents(N);
            for (int v : order) {
                const Cut &c = cuts[v][best[v]];
                for (int q = 0; q < c.n; ++q) {
                    int l = c.leaf[q];
                    bool seen = false;
                    for (int r = 0; r < q; ++r) seen |= c.leaf[r] == l;
                    if (seen || !is_gate_lut(l)) continue;
                    pend[v]++;
                    parents[l].push_back(v);
                }
            }
            std::vector<int> ready, out2;
            for (int v : order) if (pend[v] == 0) ready.push_back(v);
            const int window = atoi(getenv("ES_LIST_SCHED"));
            while (!ready.empty()) {
                int bi = -1, bs = 1 << 30, bp = 1 << 30;
                for (int i = 0; i < (int)ready.size(); ++i) {
                    const int v = ready[i];
                    const Cut &c = cuts[v][best[v]];
                    int fr = 0;
                    for (int q = 0; q < c.n; ++q) {
                        int l = c.leaf[q];
                        bool seen = false;
                        for (int r = 0; r < q; ++r) seen |= c.leaf[r] == l;
                        if (seen || !is_gate_lut(l)) continue;
                        if (rem[l] == 1) ++fr;
                    }
                    const int sc = 1 - fr;
                    // only look `window` positions ahead of the DFS order
                    if (pos[v] > (out2.empty() ? 0 : pos[out2.back()]) + window && sc >= 0) continue;
                    if (sc < bs || (sc == bs && pos[v] < bp)) { bs = sc; bp = pos[v]; bi = i; }
                }
                if (bi < 0) {  // fall back to earliest in DFS order
                    for (int i = 0; i < (int)ready.size(); ++i)
                        if (bi < 0 || pos[ready[i]] < pos[ready[bi]]) bi = i;
                }
                const int v = ready[bi];
                ready[bi] = ready.back();
                ready.pop_back();
                out2.push_back(v);
                const Cut &c = cuts[v][best[v]];
                for (int q = 0; q < c.n; ++q) {
                    int l = c.leaf[q];
                    bool seen = false;
                    for (int r = 0; r < q; ++r) seen |= c.leaf[r] == l;
                    if (seen || !is_gate_lut(l)) continue;
                    rem[l]--;
                }
                for (int pa : parents[v]) if (--pend[pa] == 0) ready.push_back(pa);
            }
            if (peak_of(out2) < peak_of(order)) order.swap(out2);
        }
    }
    // an output's inversion folds into its root LUT when nothing else reads it
    std::vector<uint8_t> out_count(N, 0), fold(N, 0);
    for (int32_t o : outs) out_count[o] = (uint8_t)std::min(2, out_count[o] + 1);
    for (size_t c = 0; c < outs.size(); ++c) {
        const int o = outs[c];
        if (is_gate_lut(o) && users[o] == 0 && out_count[o] == 1 && outs_neg[c]) {
            fold[o] = 1;
            outs_neg[c] = 0;
        }
    }
    // emit LUTs and measure the live set
    std::vector<int> remaining = users;
    for (int32_t o : outs)
        if (is_gate_lut(o)) remaining[o] += 1;
    int live = 0;
    for (int v : order) {
        const Cut &c = cuts[v][best[v]];
        Lut L{};
        L.node = v;
        L.nleaves = c.n;
        for (int q = 0; q < 3; ++q) L.leaf[q] = q < c.n ? c.leaf[q] : c.leaf[0];
        L.tt = c.tt;
        if (fold[v]) L.tt = (uint8_t)~L.tt;
        net->luts.push_back(L);
        int freed = 0;
        for (int q = 0; q < c.n; ++q) {
            int l = c.leaf[q];
            bool seen = false;
            for (int r = 0; r < q; ++r) seen |= c.leaf[r] == l;
            if (seen || !is_gate_lut(l)) continue;
            if (--remaining[l] == 0) ++freed;
        }
        live = live - freed + 1;
        net->peak_live = std::max(net->peak_live, live);
    }
    net->outs = outs;
    net->outs_neg = outs_neg;
    net->out_node = outs[0];
    net->out_neg = outs_neg[0];
}

// ---------------------------------------------------------------------------
// CPU model of the mapped program (same word layout as the kernel)
// ---------------------------------------------------------------------------
void eval_lutnet(const LutNet &net, uint64_t w0, uint64_t nw, uint32_t *out) {
    const int N = (int)net.is_const.size();
    std::vector<uint32_t> val(N, 0);
    for (int v = 0; v < N; ++v) if (net.is_const[v]) val[v] = net.const_val[v];
    const uint32_t valid = lane_valid_mask(net.num_pis);
    for (uint64_t k = 0; k < nw; ++k) {
        const uint64_t w = w0 + k;
        // w is the full word index: PI j >= 6 is bit j-6 of it, cofactor PIs
        // included -- their bits select the copy whose output is this word's
        for (int j : net.pis_used) val[j] = ((w >> (j - 6)) & 1) ? ~0u : 0u;
        for (const Lut &L : net.luts)
            val[L.node] = lut3(L.tt, val[L.leaf[2]], val[L.leaf[1]], val[L.leaf[0]]);
        int32_t c = 0;
        for (size_t b = 0; b < net.cof_pis.size(); ++b) c |= (int32_t)((w >> (net.cof_pis[b] - 6)) & 1) << b;
        size_t i = (size_t)c;  // the output of copy c (a restricted variant lacks some: 0)
        if (!net.copy_ids.empty()) {
            auto it = std::find(net.copy_ids.begin(), net.copy_ids.end(), c);
            if (it == net.copy_ids.end()) { out[k] = 0; continue; }
            i = (size_t)(it - net.copy_ids.begin());
        }
        uint32_t o = val[net.outs[i]];
        if (net.outs_neg[i]) o = ~o;
        out[k] = o & valid;
    }
}

// ---------------------------------------------------------------------------
// PTX body for the K1 skeleton
// ---------------------------------------------------------------------------
// A LUT that is a 2-input function of a word-uniform PI u (0 or ~0 for the
// whole word) and one other value x is, for each value of u, one of
// {0, ~0, x, ~x} = x*S + T with S in {0, 1, -1} and T in {0, -1}.  So it is
// one IMAD -- on the FMA pipe, idle in this kernel -- with S and T per-word
// values derived from u's bit (shared by every LUT with the same (u, S/T)
// pattern).  The ALU pipe, the kernel's bound, loses those LOP3s.
// `sel[v]`: v is word-uniform (0 or ~0 across the word) and not a constant --
// a PI >= 6 or a LUT over such nodes -- so it can act as the IMAD selector.
bool plan_imad(const Lut &L, const std::vector<uint8_t> &sel, ImadPlan *pl) {
    int vars[3], nv = 0;
    for (int k = 0; k < 3; ++k) {
        bool dep = false;
        for (int i = 0; i < 8; ++i)
            if (((L.tt >> i) & 1) != ((L.tt >> (i ^ (1 << k))) & 1)) dep = true;
        if (dep) vars[nv++] = k;
    }
    if (nv != 2 || L.leaf[vars[0]] == L.leaf[vars[1]]) return false;
    int ku = -1, kx = -1;
    if (sel[L.leaf[vars[1]]]) { ku = vars[1]; kx = vars[0]; }
    else if (sel[L.leaf[vars[0]]]) { ku = vars[0]; kx = vars[1]; }
    else return false;
    auto f = [&](int xv, int uv) { return (L.tt >> ((xv << kx) | (uv << ku))) & 1; };
    auto st = [&](int uv, int *sv, int *tv) {
        const int a = f(0, uv), b = f(1, uv);  // value at x = 0 / x = 1
        if (!a && !b) { *sv = 0; *tv = 0; }
        else if (a && b) { *sv = 0; *tv = -1; }
        else if (!a && b) { *sv = 1; *tv = 0; }
        else { *sv = -1; *tv = -1; }
    };
    st(0, &pl->s0, &pl->t0);
    st(1, &pl->s1, &pl->t1);
    pl->x = L.leaf[kx];
    pl->u = L.leaf[ku];
    return true;
}

std::string emit_body_ptx(const LutNet &net, const std::vector<std::string> &outs,
                          const std::string &wlo, const std::string &whi,
                          const std::string &one) {
    const int N = (int)net.is_const.size();
    const int P = net.num_pis;
    const bool imad = !one.empty() && getenv("ES_NO_IMAD") == nullptr;
    std::ostringstream s;
    // register names per node
    std::vector<int> lut_idx(N, -1);
    for (size_t i = 0; i < net.luts.size(); ++i) lut_idx[net.luts[i].node] = (int)i;
    std::unordered_map<uint32_t, int> cidx;
    std::vector<uint32_t> consts;
    std::vector<uint8_t> pi_mask(P + 1, 0), sel(N, 0), have_bit(N, 0);
    for (int j = 6; j <= P; ++j) sel[j] = !net.is_const[j];
    for (const Lut &L : net.luts) {
        bool u = true;
        for (int q = 0; q < 3; ++q) u = u && sel[L.leaf[q]];
        sel[L.node] = u;
    }
    auto name = [&](int v) -> std::string {
        if (lut_idx[v] >= 0) return "%esq" + std::to_string(lut_idx[v]);
        if (net.is_const[v]) {
            uint32_t c = net.const_val[v];
            auto it = cidx.find(c);
            int k;
            if (it == cidx.end()) { k = (int)consts.size(); cidx[c] = k; consts.push_back(c); }
            else k = it->second;
            return "%esk" + std::to_string(k);
        }
        pi_mask[v] = 1;
        return "%esm" + std::to_string(v);  // PI mask
    };
    std::ostringstream body;
    // per-word coefficient registers keyed by (selector, a, b) = value a at
    // u = 0, b at u = 1; emitted at first use (selectors precede their users)
    std::map<std::tuple<int, int, int>, std::string> coef;
    auto bit_of = [&](int u) {  // bit = -mask, as an IMAD by an opaque -1 (FMA pipe)
        const std::string b = "%esb" + std::to_string(u);
        if (!have_bit[u]) {
            have_bit[u] = 1;
            body << "mul.lo.s32 " << b << ", " << name(u) << ", %esneg1;\n";
        }
        return b;
    };
    auto coef_reg = [&](int u, int a, int b) -> std::string {
        if (a == b) return std::to_string(a);  // immediate
        auto key = std::make_tuple(u, a, b);
        auto it = coef.find(key);
        if (it != coef.end()) return it->second;
        const std::string r = "%esc" + std::to_string(coef.size());
        coef[key] = r;
        if (a == 0 && b == -1) {  // -bit = mask
            const std::string m = name(u);
            body << "mov.b32 " << r << ", " << m << ";\n";
        } else if (a == 0 && b == 1) {
            const std::string bt = bit_of(u);  // may emit; keep it out of the line below
            body << "mov.b32 " << r << ", " << bt << ";\n";
        } else {
            // a + (b - a) * bit = mask * (a - b) + a straight from the mask (no
            // separate bit), the factor an opaque register so the multiply
            // stays an IMAD on the FMA pipe
            const std::string m = name(u);
            const int f = a - b;  // in {-2, -1, 1, 2}
            const std::string fr = f == -1 ? "%esneg1" : f == 1 ? one : f == 2 ? "%escf2" : "%escg2";
            body << "mad.lo.s32 " << r << ", " << m << ", " << fr << ", " << a << ";\n";
        }
        return r;
    };
    // Cofactor copies: fold each copy's output into (first failing word, its
    // copy number) as soon as it exists -- 3 ops per copy, 2 live registers.
    const bool multi = net.outs.size() > 1 || !net.cof_pis.empty();
    std::vector<uint8_t> emitted(N, 0);
    size_t next_copy = 0;
    auto flush_outputs = [&]() {
        while (multi && next_copy < net.outs.size()) {
            const int o = net.outs[next_copy];
            if (lut_idx[o] >= 0 && !emitted[o]) break;
            std::string v = name(o);
            if (net.outs_neg[next_copy]) { body << "not.b32 %est, " << v << ";\n"; v = "%est"; }
            body << "setp.eq.b32 %espz, " << outs[0] << ", 0;\n"
                 << "selp.b32 " << outs[0] << ", " << v << ", " << outs[0] << ", %espz;\n"
                 << "selp.b32 " << outs[1] << ", " << net.copy_id(next_copy) << ", " << outs[1] << ", %espz;\n";
            ++next_copy;
        }
    };
    flush_outputs();
    for (const Lut &L : net.luts) {
        ImadPlan pl;
        if (imad && plan_imad(L, sel, &pl)) {
            const std::string S = coef_reg(pl.u, pl.s0, pl.s1), T = coef_reg(pl.u, pl.t0, pl.t1);
            body << "mad.lo.s32 " << name(L.node) << ", " << name(pl.x) << ", " << S << ", " << T << ";\n";
        } else {
            body << "lop3.b32 " << name(L.node) << ", " << name(L.leaf[2]) << ", " << name(L.leaf[1])
                 << ", " << name(L.leaf[0]) << ", " << (int)L.tt << ";\n";
        }
        emitted[L.node] = 1;
        flush_outputs();
    }
    std::vector<std::string> onames;
    if (!multi) onames.push_back(name(net.outs[0]));
    s << "{\n";
    if (!net.luts.empty()) s << ".reg .b32 %esq<" << net.luts.size() << ">;\n";
    if (!consts.empty()) s << ".reg .b32 %esk<" << consts.size() << ">;\n";
    s << ".reg .b32 %esm<" << (P + 1) << ">;\n.reg .b32 %esp<" << (P + 1) << ">;\n.reg .b32 %esb<" << N << ">;\n";
    if (!coef.empty()) s << ".reg .b32 %esc<" << coef.size() << ">;\n";
    for (size_t k = 0; k < consts.size(); ++k) s << "mov.b32 %esk" << k << ", " << consts[k] << ";\n";
    if (imad)
        s << ".reg .b32 %esneg1, %escf2, %escg2;\nneg.s32 %esneg1, " << one << ";\nadd.s32 %escf2, " << one << ", "
          << one << ";\nneg.s32 %escg2, %escf2;\n";
    if (multi)
        s << ".reg .pred %espz;\n.reg .b32 %est;\nmov.b32 " << outs[0] << ", 0;\nmov.b32 " << outs[1] << ", 0;\n";
    for (int j = 6; j <= P; ++j) {
        if (!pi_mask[j]) continue;
        const int bit = net.pi_bit[j];  // bit of the kernel's word index
        const std::string &src = bit < 32 ? wlo : whi;
        // (through a temporary, so every %es value has one definition: es_spill.cpp)
        if (imad) {  // mask on the FMA pipe: bit to the sign by a multiply, spread by mul.hi
            s << "mul.lo.u32 %esp" << j << ", " << src << ", " << (1u << (31 - (bit & 31))) << ";\n";
            s << "mul.hi.s32 %esm" << j << ", %esp" << j << ", " << one << ";\n";
        } else {
            s << "shl.b32 %esp" << j << ", " << src << ", " << (31 - (bit & 31)) << ";\n";
            s << "shr.s32 %esm" << j << ", %esp" << j << ", 31;\n";
        }
    }
    s << body.str();
    if (!multi)
        s << (net.outs_neg[0] ? "not.b32 " : "mov.b32 ") << outs[0] << ", " << onames[0] << ";\n";
    s << "}\n";
    return s.str();
}


}  // namespace es
