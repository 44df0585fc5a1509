// es_k2prog.cpp -- program format of K2, the shared-memory interpreter.
//
// K2 runs programs that are not worth a JIT (small sweeps, batches of
// thousands of cones).  Its cost is shared-memory traffic per gate, so the
// host re-schedules the reference program (any InstrProgram, es.py:66-73) for
// it instead of interpreting the reference order verbatim:
//   * gate-level DFS post-order with children by decreasing register need, so
//     most gates consume the previous gate's result;
//   * that operand (always operand A) is read from an accumulator register
//     (no LDS; a non-accumulator A is loaded straight into it), and a result
//     whose only consumers are the next gate's operand A and the outputs
//     folded right after it is never stored (no STS);
//   * the remaining live values get LIFO-recycled slots after the PI slots
//     (fanins are freed before the destination is allocated, as es.py:151-156);
//   * complement flags become record bits; XOR folds both into operand A's.
// Cofactor copies (es_cofactor.cpp): the graph may have 2^k outputs, one per
// assignment of k word PIs that are then fixed per copy instead of per word;
// OUT records fold each copy's output into (first failing word, copy number)
// in copy order, so the kernel's rare path can rebuild the minimum index.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <queue>
#include <tuple>

#include "es_k2prog.h"

namespace es {

namespace {

struct Outs {
    std::vector<int32_t> node;
    std::vector<uint8_t> neg;
};

Outs outputs_of(const Dag &dag) {
    Outs o;
    if (dag.outs.empty()) { o.node.push_back(dag.out_node); o.neg.push_back(dag.out_neg); }
    else { o.node = dag.outs; o.neg = dag.outs_neg; }
    return o;
}

void emit_k2(const Dag &dag, const Outs &outs, const std::vector<int> &order,
             const std::vector<uint8_t> &cone, std::vector<int> refs, K2Prog *kp) {
    const int N = dag.num_nodes(), FG = dag.first_gate(), P = dag.num_pis;
    auto is_gate = [&](int v) { return v >= FG && cone[v]; };
    kp->num_pis = P;
    kp->gates.clear();
    kp->n_gates = 0;
    kp->loads = kp->stores = 0;
    // slots: 0..P-1 hold the PI words (filled once per word batch); gates
    // above, LIFO-recycled
    std::vector<int> slot(N, -1), pool, pos(N, -1);
    for (int j = 1; j <= P; ++j) slot[j] = j - 1;
    for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = (int)i;
    int top = P;
    auto alloc = [&]() {
        if (!pool.empty()) { int s = pool.back(); pool.pop_back(); return s; }
        return top++;
    };
    // each copy's output is folded as soon as it exists and after the previous
    // copy's: flush position = max(previous, position of its node)
    const int C = (int)outs.node.size();
    std::vector<int> flush(C, -1);
    for (int c = 0; c < C; ++c) {
        const int o = outs.node[c];
        flush[c] = std::max(c ? flush[c - 1] : -1, is_gate(o) ? pos[o] : -1);
    }
    int next_copy = 0;
    int last_gate = -1;  // node in the accumulator
    auto emit_outs = [&](int upto) {
        for (; next_copy < C && flush[next_copy] <= upto; ++next_copy) {
            const int o = outs.node[next_copy];
            const bool neg = outs.neg[next_copy];
            K2Gate g{};
            uint32_t ctl = K2_OUT | ((uint32_t)next_copy << 16) | (neg ? K2_NEG_A : 0u);
            if (o == 0) {
                if (!neg) continue;  // constant 0: this copy never fails
                ctl |= K2_CONST;
            } else if (o == last_gate) {
                ctl |= K2_A_ACC;
            } else {
                g.a = (uint32_t)slot[o];
                kp->loads++;
            }
            g.ctl = ctl;
            kp->gates.push_back(g);
            if (is_gate(o) && --refs[o] == 0 && slot[o] >= P) pool.push_back(slot[o]);
        }
    };
    emit_outs(-1);
    for (size_t i = 0; i < order.size(); ++i) {
        const int v = order[i], gi = v - FG;
        int fa = dag.f0[gi], fb = dag.f1[gi];
        uint32_t na = dag.n0[gi], nb = dag.n1[gi];
        // only operand A may come from the accumulator: swap the previous
        // gate's result into A (AND and XOR are symmetric)
        if (fb == last_gate && fa != last_gate) { std::swap(fa, fb); std::swap(na, nb); }
        K2Gate g{};
        uint32_t ctl = dag.is_xor[gi] ? K2_XOR : 0u;
        if (fa == last_gate) ctl |= K2_A_ACC;
        else { g.a = (uint32_t)slot[fa]; kp->loads++; }
        g.b = (uint32_t)slot[fb];  // == last_gate only for AND(x, x): then x was stored
        kp->loads++;
        if (dag.is_xor[gi]) { if (na ^ nb) ctl |= K2_NEG_A; }
        else { if (na) ctl |= K2_NEG_A; if (nb) ctl |= K2_NEG_B; }
        // consume fanins; a slot frees when its last reader has read it
        for (int f : {fa, fb}) {
            if (!is_gate(f)) continue;
            if (--refs[f] == 0 && slot[f] >= 0) pool.push_back(slot[f]);
        }
        // readers served by the accumulator: outputs folded right after this
        // gate, and operand A of the next gate
        int acc_uses = 0;
        for (int c = next_copy; c < C && flush[c] == (int)i; ++c) acc_uses += outs.node[c] == v;
        if (i + 1 < order.size()) {
            const int nx = order[i + 1] - FG;
            const bool a_ = dag.f0[nx] == v, b_ = dag.f1[nx] == v;
            acc_uses += (a_ != b_) ? 1 : 0;
        }
        if (refs[v] > acc_uses) {
            ctl |= K2_STORE;
            slot[v] = alloc();
            g.d = (uint32_t)slot[v];
            kp->stores++;
        }
        g.ctl = ctl;
        kp->gates.push_back(g);
        kp->n_gates++;
        last_gate = v;
        emit_outs((int)i);
    }
    kp->num_slots = top;
}

// Multi-lane program (K2Prog::lanes = L > 1): an L-processor list schedule
// of `order` -- each step takes up to L gates that are all ready (so none
// reads another of the same step), preferring for each lane a gate that
// consumes that lane's previous result (served by the lane's accumulator),
// within a window of the order so the live set stays close to the
// sequential schedule's.  The interpreter then has L independent dependency
// chains per warp.  Outputs fold in copy order in OUT steps of up to L
// records.
static int k2_window() {  // window 4: 15.3 ms, 8: 14.0, 16: 13.6, 32: 13.8, 64: 15.3 (first two-lane kernel)
    static const int w = getenv("ES_K2_LANE_WIN") ? std::max(2, atoi(getenv("ES_K2_LANE_WIN"))) : 16;
    return w;
}

}  // namespace

int k2_lanes() {
    static const int L = [] {
        // two lanes by default: config 4 15.9 -> 11.9 ms on the B200 (one
        // lane: latency-bound, stall_wait 2.2 per issue; four: 12.2 ms, NOP
        // lanes and OUT padding cost more than the extra ILP gains)
        const char *e = getenv("ES_K2_LANES");
        const int v = e ? atoi(e) : 2;
        return v >= 4 ? 4 : v >= 2 ? 2 : 1;
    }();
    return L;
}

namespace {

void emit_k2_lanes(const Dag &dag, const Outs &outs, const std::vector<int> &order,
                   const std::vector<uint8_t> &cone, int L, K2Prog *kp) {
    const int N = dag.num_nodes(), FG = dag.first_gate(), P = dag.num_pis;
    auto is_gate = [&](int v) { return v >= FG && cone[v]; };
    const int n = (int)order.size(), C = (int)outs.node.size();
    struct Step { int g[4] = {-1, -1, -1, -1}; int out0 = -1, nout = 0; };
    std::vector<Step> steps;
    std::vector<int> step_of(N, -1);
    std::vector<int8_t> lane_of(N, -1);
    std::vector<uint8_t> done(N, 0);
    auto ready = [&](int v) {
        const int g = v - FG;
        return (!is_gate(dag.f0[g]) || done[dag.f0[g]]) && (!is_gate(dag.f1[g]) || done[dag.f1[g]]);
    };
    auto reads = [&](int v, int u) {
        const int g = v - FG;
        return u >= 0 && (dag.f0[g] == u || dag.f1[g] == u);
    };
    int next_copy = 0;
    auto flush = [&]() {
        while (next_copy < C) {
            const int o = outs.node[next_copy];
            if (is_gate(o) && !done[o]) break;
            if (steps.empty() || steps.back().out0 < 0 || steps.back().nout == L) {
                Step st;
                st.out0 = next_copy;
                steps.push_back(st);
            }
            steps.back().nout++;
            ++next_copy;
        }
    };
    flush();
    int first = 0, last[4] = {-1, -1, -1, -1};
    std::vector<int> cand;
    for (int scheduled = 0; scheduled < n;) {
        while (first < n && done[order[first]]) ++first;
        cand.clear();
        for (int i = first; i < n && i < first + k2_window(); ++i)
            if (!done[order[i]] && ready(order[i])) cand.push_back(order[i]);
        // (order[first] is always ready: `order` is topological)
        int pick[4] = {-1, -1, -1, -1};
        auto taken = [&](int v) {
            for (int h = 0; h < L; ++h) if (pick[h] == v) return true;
            return false;
        };
        for (int h = 0; h < L; ++h)
            for (int v : cand)
                if (!taken(v) && reads(v, last[h])) { pick[h] = v; break; }
        for (int h = 0; h < L; ++h)
            if (pick[h] < 0)
                for (int v : cand)
                    if (!taken(v)) { pick[h] = v; break; }
        Step st;
        for (int h = 0; h < L; ++h) {
            const int v = pick[h];
            if (v < 0) continue;
            st.g[h] = v;
            done[v] = 1;
            step_of[v] = (int)steps.size();
            lane_of[v] = (int8_t)h;
            last[h] = v;
            ++scheduled;
        }
        steps.push_back(st);
        flush();
    }
    // the next gate of each gate's lane: its accumulator holds the gate's
    // value until then
    std::vector<int> nxt(N, -1);
    {
        int prev[4] = {-1, -1, -1, -1};
        for (const Step &st : steps)
            for (int h = 0; h < L; ++h)
                if (st.g[h] >= 0) {
                    if (prev[h] >= 0) nxt[prev[h]] = st.g[h];
                    prev[h] = st.g[h];
                }
    }
    auto by_acc = [&](int reader, int f) {  // gate `reader` gets gate f from the accumulator
        return is_gate(f) && lane_of[f] == lane_of[reader] && nxt[f] == reader;
    };
    auto out_by_acc = [&](int step, int o) {
        return is_gate(o) && (nxt[o] < 0 || step_of[nxt[o]] > step);
    };
    // slot readers of every value (one per reader, however many operands)
    std::vector<int> sref(N, 0);
    for (size_t si = 0; si < steps.size(); ++si) {
        const Step &st = steps[si];
        if (st.out0 >= 0) {
            for (int c = st.out0; c < st.out0 + st.nout; ++c) {
                const int o = outs.node[c];
                if (o != 0 && !out_by_acc((int)si, o)) sref[o]++;
            }
            continue;
        }
        for (int h = 0; h < L; ++h) {
            const int v = st.g[h];
            if (v < 0) continue;
            const int g = v - FG, fa = dag.f0[g], fb = dag.f1[g];
            if (fa == fb) { sref[fa]++; continue; }  // g(x, x): B from x's slot (A maybe from the accumulator)
            // one operand may come from the accumulator (swapped into A)
            const bool aa = by_acc(v, fa), ab = !aa && by_acc(v, fb);
            if (!aa) sref[fa]++;
            if (!ab) sref[fb]++;
        }
    }
    kp->num_pis = P;
    kp->gates.clear();
    kp->n_gates = 0;
    kp->loads = kp->stores = 0;
    kp->lanes = L;
    // slots: the PI words, then one slot the kernel zeroes (a NOP lane is
    // acc & ~0 over it), then the gates, LIFO-recycled
    std::vector<int> slot(N, -1), pool;
    for (int j = 1; j <= P; ++j) slot[j] = j - 1;
    int top = P + 1;
    auto alloc = [&]() {
        if (!pool.empty()) { int q = pool.back(); pool.pop_back(); return q; }
        return top++;
    };
    auto release = [&](int v) {
        if (is_gate(v) && --sref[v] == 0 && slot[v] > P) pool.push_back(slot[v]);
    };
    const K2Gate nop{0u, (uint32_t)P, 0u, K2_A_ACC | K2_NEG_B};
    for (size_t si = 0; si < steps.size(); ++si) {
        const Step &st = steps[si];
        if (st.out0 >= 0) {
            std::vector<K2Gate> rec;
            for (int c = st.out0; c < st.out0 + st.nout; ++c) {
                const int o = outs.node[c];
                const bool neg = outs.neg[c];
                K2Gate g{};
                uint32_t ctl = K2_OUT | ((uint32_t)c << 16) | (neg ? K2_NEG_A : 0u);
                if (o == 0) {
                    if (!neg) continue;  // constant 0: this copy never fails
                    ctl |= K2_CONST;
                } else if (out_by_acc((int)si, o)) {
                    ctl |= K2_A_ACC | ((uint32_t)lane_of[o] << K2_OUT_LANE_SHIFT);
                } else {
                    g.a = (uint32_t)slot[o];
                    kp->loads++;
                }
                g.ctl = ctl;
                rec.push_back(g);
                if (o != 0 && !(ctl & K2_A_ACC)) release(o);
            }
            if (rec.empty()) continue;
            while ((int)rec.size() < L) rec.push_back(nop);  // (no K2_OUT: skipped by the OUT step)
            kp->gates.insert(kp->gates.end(), rec.begin(), rec.end());
            continue;
        }
        K2Gate rec[4] = {nop, nop, nop, nop};
        std::vector<int> reads_from_slot;
        for (int h = 0; h < L; ++h) {
            const int v = st.g[h];
            if (v < 0) continue;
            const int gi = v - FG;
            int fa = dag.f0[gi], fb = dag.f1[gi];
            uint32_t na = dag.n0[gi], nb = dag.n1[gi];
            if (fa != fb && !by_acc(v, fa) && by_acc(v, fb)) { std::swap(fa, fb); std::swap(na, nb); }
            K2Gate g{};
            uint32_t ctl = dag.is_xor[gi] ? K2_XOR : 0u;
            if (by_acc(v, fa)) ctl |= K2_A_ACC;
            else { g.a = (uint32_t)slot[fa]; kp->loads++; }
            g.b = (uint32_t)slot[fb];  // (g(x, x): x was stored; a step's loads follow the last step's stores)
            kp->loads++;
            if (dag.is_xor[gi]) { if (na ^ nb) ctl |= K2_NEG_A; }
            else { if (na) ctl |= K2_NEG_A; if (nb) ctl |= K2_NEG_B; }
            g.ctl = ctl;
            rec[h] = g;
            if (fa == fb) reads_from_slot.push_back(fa);  // one reader of x
            else {
                if (!(ctl & K2_A_ACC)) reads_from_slot.push_back(fa);
                reads_from_slot.push_back(fb);
            }
            kp->n_gates++;
        }
        // every lane has read: free the slots whose last reader this step was,
        // then place the results (a step's stores follow its loads)
        for (int f : reads_from_slot) release(f);
        for (int h = 0; h < L; ++h) {
            const int v = st.g[h];
            if (v < 0 || sref[v] == 0) continue;
            slot[v] = alloc();
            rec[h].d = (uint32_t)slot[v];
            rec[h].ctl |= K2_STORE;
            kp->stores++;
        }
        for (int h = 0; h < L; ++h) {
            if (st.g[h] < 0) kp->loads++;  // a NOP lane still loads the zero slot
            kp->gates.push_back(rec[h]);
        }
    }
    // every gate record of a multi-lane step stores (es_k2d has no store
    // test): results nobody reads, and the NOP lanes', go to one dummy slot
    const int dummy = top++;
    for (K2Gate &g : kp->gates)
        if (!(g.ctl & K2_OUT) && !(g.ctl & K2_STORE)) {
            g.d = (uint32_t)dummy;
            kp->stores++;
        }
    kp->num_slots = top;
}

}  // namespace

void build_k2prog(const Dag &dag, K2Prog *kp) {
    const int N = dag.num_nodes(), FG = dag.first_gate(), P = dag.num_pis;
    const Outs outs = outputs_of(dag);
    std::vector<uint8_t> cone(N, 0);
    for (int32_t o : outs.node) cone[o] = 1;
    for (int v = N - 1; v >= FG; --v) {
        if (!cone[v]) continue;
        cone[dag.f0[v - FG]] = cone[dag.f1[v - FG]] = 1;
    }
    auto is_gate = [&](int v) { return v >= FG && cone[v]; };
    // register need, bottom-up; references (outputs count once per copy)
    std::vector<int> need(N, 0), refs(N, 0);
    for (int32_t o : outs.node) refs[o] += 1;
    for (int v = FG; v < N; ++v) {
        if (!cone[v]) continue;
        const int g = v - FG, a = dag.f0[g], b = dag.f1[g];
        refs[a]++; refs[b]++;
        int na = is_gate(a) ? need[a] : 0, nb = is_gate(b) ? need[b] : 0;
        if (na < nb) std::swap(na, nb);
        need[v] = std::max({1, na, nb + 1});
    }
    // candidate 1: DFS post-order from each output in copy order, highest-need child first
    std::vector<int> order;
    {
        std::vector<uint8_t> done(N, 0);
        std::vector<int> st;
        for (int32_t o : outs.node) {
            if (!is_gate(o) || done[o]) continue;
            st.push_back(o);
            while (!st.empty()) {
                const int v = st.back();
                if (done[v]) { st.pop_back(); continue; }
                const int g = v - FG;
                int pick = -1;
                for (int l : {dag.f0[g], dag.f1[g]})
                    if (is_gate(l) && !done[l] && (pick < 0 || need[l] > need[pick])) pick = l;
                if (pick >= 0) { st.push_back(pick); continue; }
                done[v] = 1;
                order.push_back(v);
                st.pop_back();
            }
        }
    }
    // candidate 2: topological (node index) order -- the reference's
    std::vector<int> topo;
    for (int v = FG; v < N; ++v)
        if (cone[v]) topo.push_back(v);
    // candidate 3: greedy list schedule -- among the ready gates, the one that
    // frees the most live values (ties: earliest in the DFS order); on wide
    // cofactored graphs it needs far fewer slots than the DFS
    std::vector<int> lsched;
    {
        std::vector<int> dpos(N, 0), pend(N, 0), rem = refs;
        for (size_t i = 0; i < order.size(); ++i) dpos[order[i]] = (int)i;
        // readers of each gate, CSR (ustart[l]..ustart[l+1]); a gate reading
        // the same fanin twice is one reader
        std::vector<int> ustart(N + 1, 0), uidx;
        for (int v : order) {
            const int g = v - FG;
            if (is_gate(dag.f0[g])) ustart[dag.f0[g] + 1]++;
            if (dag.f1[g] != dag.f0[g] && is_gate(dag.f1[g])) ustart[dag.f1[g] + 1]++;
        }
        for (int v = 0; v < N; ++v) ustart[v + 1] += ustart[v];
        uidx.resize(ustart[N]);
        {
            std::vector<int> fill(ustart.begin(), ustart.end() - 1);
            for (int v : order) {
                const int g = v - FG;
                for (int l : {dag.f0[g], dag.f1[g]}) {
                    if (!is_gate(l)) continue;
                    if (dag.f0[g] == dag.f1[g] && l == dag.f1[g] && pend[v]) continue;
                    pend[v]++;
                    uidx[fill[l]++] = v;
                }
            }
        }
        struct Users {
            const int *b, *e;
            const int *begin() const { return b; }
            const int *end() const { return e; }
        };
        auto users = [&](int l) { return Users{uidx.data() + ustart[l], uidx.data() + ustart[l + 1]}; };
        // lazy min-heap of (score, DFS position, gate); scores only improve
        // as fanins lose readers, so stale entries are skipped on pop
        auto score = [&](int v) {
            const int g = v - FG, a0 = dag.f0[g], a1 = dag.f1[g];
            int fr = 0;
            if (is_gate(a0) && rem[a0] == (a0 == a1 ? 2 : 1)) ++fr;
            if (a1 != a0 && is_gate(a1) && rem[a1] == 1) ++fr;
            return 1 - fr;
        };
        using E = std::tuple<int, int, int>;
        std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
        std::vector<uint8_t> in_ready(N, 0), done(N, 0);
        for (int v : order)
            if (pend[v] == 0) { in_ready[v] = 1; heap.emplace(score(v), dpos[v], v); }
        while (!heap.empty()) {
            const auto [sc, dp, v] = heap.top();
            heap.pop();
            if (done[v] || sc != score(v)) continue;
            done[v] = 1;
            lsched.push_back(v);
            const int g = v - FG;
            for (int l : {dag.f0[g], dag.f1[g]}) {
                if (!is_gate(l)) continue;
                rem[l]--;
                if (rem[l] <= 2)  // a remaining ready reader may now free l
                    for (int u : users(l))
                        if (in_ready[u] && !done[u]) heap.emplace(score(u), dpos[u], u);
            }
            for (int u : users(v))
                if (--pend[u] == 0) { in_ready[u] = 1; heap.emplace(score(u), dpos[u], u); }
        }
    }
    // the list schedule needs about half the slots of the DFS on cofactored
    // graphs (and wins on ~98 % of the config-4 cones); the reference order
    // still wins now and then on single-output programs
    if (k2_lanes() > 1) {
        emit_k2_lanes(dag, outs, lsched, cone, k2_lanes(), kp);
        return;
    }
    emit_k2(dag, outs, lsched, cone, refs, kp);
    if (outs.node.size() == 1) {
        K2Prog b;
        emit_k2(dag, outs, topo, cone, refs, &b);
        auto cost = [](const K2Prog &q) { return std::make_pair(q.num_slots, q.loads + q.stores); };
        if (cost(b) < cost(*kp)) *kp = std::move(b);
    }
}

void build_k2prog_k(const Dag &dag, int k, K2Prog *kp) {
    if (k <= 0) { build_k2prog(dag, kp); kp->cof_pis.clear(); return; }
    std::vector<int32_t> pis = rank_cofactor_pis(dag, k);
    std::sort(pis.begin(), pis.end());
    Dag x;
    cofactor_expand(dag, pis, &x);
    build_k2prog(x, kp);
    kp->cof_pis = pis;
}

void build_k2prog_auto(const Dag &dag, K2Prog *kp, int min_words_log2, int max_slots,
                       double min_work) {
    if (const char *e = getenv("ES_K2_MAXSLOTS")) max_slots = atoi(e);
    const int P = dag.num_pis;
    int kmax = std::min(kK2MaxCofactorPis, P - 5 - min_words_log2);
    if ((double)dag.is_xor.size() * std::ldexp(1.0, P) < min_work) kmax = 0;
    std::vector<int32_t> rank;
    if (kmax >= 1) rank = rank_cofactor_pis(dag, kmax);
    // gates per word of each depth (the interpreter's cost is ~linear in the
    // gate count); the expansions share copy 0's literals outside the
    // cofactor PIs' fanout, so they are cheap.  Build the best depth, and
    // step down while its program needs more slots than the budget.
    std::vector<Dag> xs(rank.size() + 1);
    std::vector<double> per_word(rank.size() + 1, 0.0);
    int gates0 = 0;
    for (int v = 0; v < (int)dag.is_xor.size(); ++v) gates0++;
    per_word[0] = (double)gates0;
    for (int k = 1; k <= (int)rank.size(); ++k) {
        std::vector<int32_t> pis(rank.begin(), rank.begin() + k);
        std::sort(pis.begin(), pis.end());
        cofactor_expand(dag, pis, &xs[k]);
        per_word[k] = (double)xs[k].is_xor.size() / (double)(1u << k) + 0.25;  // + OUT records
    }
    std::vector<int> order(per_word.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = (int)k;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return per_word[a] < per_word[b]; });
    // The cheapest depth by gates may need > 88 slots, which the runtime runs
    // at one word per thread (W=1, two CTAs per SM when it fits), so weigh
    // occupancy: also try the next depths until one fits 88 slots and keep
    // the lower effective cost.  Penalties re-measured on config 4 after the
    // K2 tuning (big 1.5: 22.4 ms, 2: 21.3, 2.5: 19.1, 3: 20.0, 3.5: 20.0;
    // mid 1.1 vs 1.25-1.6 within noise or worse).
    static const double big_pen = getenv("ES_K2_BIGPEN") ? atof(getenv("ES_K2_BIGPEN")) : 2.5;
    static const double mid_pen = getenv("ES_K2_MIDPEN") ? atof(getenv("ES_K2_MIDPEN")) : 1.1;
    auto occupancy_cost = [](const K2Prog &q, double pw) {
        const int g = k2_group_of(q.num_slots, k2_device_records(q));
        return pw * (g == 2 ? big_pen : g == 1 ? mid_pen : 1.0);
    };
    bool have = false;
    double best = 0;
    int builds = 0;
    for (int k : order) {
        K2Prog q;
        if (k == 0) build_k2prog(dag, &q);
        else build_k2prog(xs[k], &q);
        ++builds;
        // over 88 slots the runtime runs one word per thread at two CTAs per SM
        // only if slots + staged records fit half an SM's shared memory
        // (2 x (smem + 1 KB reserve + statics) <= 228 KB); otherwise one 4-warp CTA, which
        // measured 12 % slower on config 4 than capping the depth
        const size_t w1_smem = (size_t)q.num_slots * 128 * 4 + (k2_device_records(q) + kK2PadRecords) * 16;
        const bool fits = q.num_slots <= max_slots && (k2_group_of(q.num_slots, k2_device_records(q)) < 2 ||
                                                       w1_smem <= kK2TwoCtaBytes);
        if (!fits && k != 0) continue;
        const double c = occupancy_cost(q, per_word[k]);
        if (!have || c < best) {
            q.cof_pis.assign(rank.begin(), rank.begin() + k);
            std::sort(q.cof_pis.begin(), q.cof_pis.end());
            *kp = std::move(q);
            best = c;
            have = true;
        }
        if (k2_group_of(kp->num_slots, k2_device_records(*kp)) < 2 || builds >= 4 || k == 0) break;
    }
}

static void eval_k2prog_lanes(const K2Prog &kp, uint64_t w0, uint64_t nw, uint32_t *out) {
    static const uint32_t lane[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
    const int L = kp.lanes;
    std::vector<uint32_t> s(std::max(kp.num_slots, 1), 0);
    const int C = 1 << kp.cof_pis.size();
    std::vector<uint32_t> val(C, 0);
    const uint32_t valid = lane_valid_mask(kp.num_pis);
    for (uint64_t k = 0; k < nw; ++k) {
        const uint64_t w = w0 + k;
        for (int j = 0; j < kp.num_pis; ++j)
            s[j] = j < 5 ? lane[j] : (((w >> (j - 5)) & 1) ? ~0u : 0u);
        std::fill(val.begin(), val.end(), 0u);
        if (kp.num_slots > kp.num_pis) s[kp.num_pis] = 0u;  // the NOP lanes' zero slot
        uint32_t acc[4] = {0, 0, 0, 0};
        for (size_t i = 0; i + L <= kp.gates.size(); i += L) {
            if (kp.gates[i].ctl & K2_OUT) {  // OUT step: fold in record (copy) order
                for (int h = 0; h < L; ++h) {
                    const K2Gate &x = kp.gates[i + h];
                    if (!(x.ctl & K2_OUT)) continue;
                    const uint32_t ma = (x.ctl & K2_NEG_A) ? ~0u : 0u;
                    const uint32_t v = (x.ctl & K2_CONST) ? 0u
                                     : (x.ctl & K2_A_ACC) ? acc[(x.ctl >> K2_OUT_LANE_SHIFT) & 3u] : s[x.a];
                    val[(x.ctl >> 16) & 0x3FFFu] = v ^ ma;
                }
                continue;
            }
            uint32_t r[4];
            for (int h = 0; h < L; ++h) {  // every lane reads before any stores
                const K2Gate &g = kp.gates[i + h];
                const uint32_t ma = (g.ctl & K2_NEG_A) ? ~0u : 0u, mb = (g.ctl & K2_NEG_B) ? ~0u : 0u;
                const uint32_t a = (g.ctl & K2_A_ACC) ? acc[h] : s[g.a];
                const uint32_t b = s[g.b];
                r[h] = (g.ctl & K2_XOR) ? (a ^ b ^ ma) : ((a ^ ma) & (b ^ mb));
            }
            for (int h = 0; h < L; ++h) {
                const K2Gate &g = kp.gates[i + h];
                if (g.ctl & K2_STORE) s[g.d] = r[h];
                acc[h] = r[h];
            }
        }
        size_t c = 0;
        for (size_t b = 0; b < kp.cof_pis.size(); ++b) c |= (size_t)((w >> (kp.cof_pis[b] - 6)) & 1) << b;
        out[k] = val[c] & valid;
    }
}

void eval_k2prog(const K2Prog &kp, uint64_t w0, uint64_t nw, uint32_t *out) {
    if (kp.lanes > 1) { eval_k2prog_lanes(kp, w0, nw, out); return; }
    static const uint32_t lane[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
    std::vector<uint32_t> s(std::max(kp.num_slots, 1), 0);
    const int C = 1 << kp.cof_pis.size();
    std::vector<uint32_t> val(C, 0);
    const uint32_t valid = lane_valid_mask(kp.num_pis);
    for (uint64_t k = 0; k < nw; ++k) {
        const uint64_t w = w0 + k;
        for (int j = 0; j < kp.num_pis; ++j)
            s[j] = j < 5 ? lane[j] : (((w >> (j - 5)) & 1) ? ~0u : 0u);
        std::fill(val.begin(), val.end(), 0u);
        uint32_t acc = 0;
        for (const K2Gate &g : kp.gates) {
            const uint32_t ma = (g.ctl & K2_NEG_A) ? ~0u : 0u, mb = (g.ctl & K2_NEG_B) ? ~0u : 0u;
            if (g.ctl & K2_OUT) {
                const uint32_t v = (g.ctl & K2_CONST) ? 0u : (g.ctl & K2_A_ACC) ? acc : s[g.a];
                val[g.ctl >> 16] = v ^ ma;
                continue;
            }
            const uint32_t a = (g.ctl & K2_A_ACC) ? acc : s[g.a];
            const uint32_t b = s[g.b];
            const uint32_t r = (g.ctl & K2_XOR) ? (a ^ b ^ ma) : ((a ^ ma) & (b ^ mb));
            if (g.ctl & K2_STORE) s[g.d] = r;
            acc = r;
        }
        size_t c = 0;
        for (size_t b = 0; b < kp.cof_pis.size(); ++b) c |= (size_t)((w >> (kp.cof_pis[b] - 6)) & 1) << b;
        out[k] = val[c] & valid;
    }
}

}  // namespace es
