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
//     whose only consumer is the next gate is never stored (no STS);
//   * the remaining live values get LIFO-recycled slots after the PI slots
//     (fanins are freed before the destination is allocated, as es.py:151-156);
//   * complement flags become full-word masks; XOR folds both into one mask.
#include <algorithm>
#include <functional>

#include "es_k2prog.h"

namespace es {

static void emit_k2(const Dag &dag, const std::vector<int> &order, const std::vector<uint8_t> &cone,
                    std::vector<int> refs, K2Prog *kp);

void build_k2prog(const Dag &dag, K2Prog *kp) {
    const int N = dag.num_nodes(), FG = dag.first_gate(), P = dag.num_pis;
    kp->num_pis = P;
    kp->gates.clear();
    kp->out_mask = dag.out_neg ? ~0u : 0u;
    kp->const_out = false;
    if (dag.out_node == 0) {  // constant output (callers normally short-cut it)
        kp->const_out = true;
        kp->num_slots = P;
        return;
    }
    std::vector<uint8_t> cone(N, 0);
    cone[dag.out_node] = 1;
    for (int v = N - 1; v >= FG; --v) {
        if (!cone[v]) continue;
        cone[dag.f0[v - FG]] = cone[dag.f1[v - FG]] = 1;
    }
    auto is_gate = [&](int v) { return v >= FG && cone[v]; };
    // register need, bottom-up
    std::vector<int> need(N, 0), refs(N, 0);
    refs[dag.out_node] += 1;
    for (int v = FG; v < N; ++v) {
        if (!cone[v]) continue;
        const int g = v - FG, a = dag.f0[g], b = dag.f1[g];
        refs[a]++; refs[b]++;
        int na = is_gate(a) ? need[a] : 0, nb = is_gate(b) ? need[b] : 0;
        if (na < nb) std::swap(na, nb);
        need[v] = std::max({1, na, nb + 1});
    }
    // DFS post-order from the output, highest-need child first
    std::vector<int> order;
    if (is_gate(dag.out_node)) {
        std::vector<uint8_t> done(N, 0);
        std::vector<int> st{dag.out_node};
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
    // candidate 2: the reference's topological order (node index order)
    std::vector<int> topo;
    for (int v = FG; v < N; ++v)
        if (cone[v]) topo.push_back(v);
    K2Prog a, b;
    a.num_pis = b.num_pis = P;
    a.out_mask = b.out_mask = kp->out_mask;
    emit_k2(dag, order, cone, refs, &a);
    emit_k2(dag, topo, cone, refs, &b);
    auto cost = [](const K2Prog &q) {
        int st = 0, acc = 0;
        for (const K2Gate &g : q.gates) { st += (g.ctl & K2_STORE) != 0; acc += ((g.ctl & K2_A_ACC) != 0) + ((g.ctl & K2_B_ACC) != 0); }
        return std::make_pair(q.num_slots, st - acc);
    };
    *kp = cost(a) <= cost(b) ? std::move(a) : std::move(b);
}

static void emit_k2(const Dag &dag, const std::vector<int> &order, const std::vector<uint8_t> &cone,
                    std::vector<int> refs, K2Prog *kp) {
    const int N = dag.num_nodes(), FG = dag.first_gate(), P = dag.num_pis;
    auto is_gate = [&](int v) { return v >= FG && cone[v]; };
    // slots: 0..P-1 hold the PI words (filled once per word batch); gates
    // above, LIFO-recycled
    std::vector<int> slot(N, -1), pool;
    for (int j = 1; j <= P; ++j) slot[j] = j - 1;
    int top = P;
    auto alloc = [&]() {
        if (!pool.empty()) { int s = pool.back(); pool.pop_back(); return s; }
        return top++;
    };
    if (order.empty()) {  // output is a PI: out = AND(pi, pi)
        K2Gate g{};
        g.a = g.b = (uint32_t)slot[dag.out_node];
        g.ma = g.mb = 0;
        g.ctl = 0;
        kp->gates.push_back(g);
        kp->num_slots = P;
        return;
    }
    for (size_t i = 0; i < order.size(); ++i) {
        const int v = order[i], gi = v - FG;
        const int prev = i > 0 ? order[i - 1] : -1;
        int fa = dag.f0[gi], fb = dag.f1[gi];
        uint32_t na = dag.n0[gi], nb = dag.n1[gi];
        // only operand A may come from the accumulator: swap a previous-gate
        // operand into A (AND and XOR are symmetric)
        if (fb == prev && fa != prev) { std::swap(fa, fb); std::swap(na, nb); }
        K2Gate g{};
        uint32_t ctl = dag.is_xor[gi] ? K2_XOR : 0u;
        if (fa == prev) ctl |= K2_A_ACC; else g.a = (uint32_t)slot[fa];
        g.b = (uint32_t)slot[fb];  // == prev only for AND(x, x): then x was stored
        const uint32_t ma = na ? ~0u : 0u, mb = nb ? ~0u : 0u;
        if (dag.is_xor[gi]) { g.ma = ma ^ mb; g.mb = 0; }
        else { g.ma = ma; g.mb = mb; }
        // consume fanins; a slot frees when its last reader has read it
        for (int f : {fa, fb}) {
            if (!is_gate(f)) continue;
            if (--refs[f] == 0 && slot[f] >= 0) pool.push_back(slot[f]);
        }
        // store unless the only remaining use is operand A of the next gate
        // (or the output, which reads the accumulator after the last gate)
        const int next = i + 1 < order.size() ? order[i + 1] : -1;
        const int next_uses = next < 0 ? 1 : ((dag.f0[next - FG] == v || dag.f1[next - FG] == v) ? 1 : 0);
        if (refs[v] > next_uses) {
            ctl |= K2_STORE;
            slot[v] = alloc();
            g.d = (uint32_t)slot[v];
        }
        g.ctl = ctl;
        kp->gates.push_back(g);
    }
    kp->num_slots = top;
}

void eval_k2prog(const K2Prog &kp, uint64_t w0, uint64_t nw, uint32_t *out) {
    static const uint32_t lane[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
    std::vector<uint32_t> s(std::max(kp.num_slots, 1), 0);
    const uint32_t valid = lane_valid_mask(kp.num_pis);
    for (uint64_t k = 0; k < nw; ++k) {
        const uint64_t w = w0 + k;
        if (kp.const_out) { out[k] = kp.out_mask & valid; continue; }
        for (int j = 0; j < kp.num_pis; ++j)
            s[j] = j < 5 ? lane[j] : (((w >> (j - 5)) & 1) ? ~0u : 0u);
        uint32_t acc = 0;
        for (const K2Gate &g : kp.gates) {
            const uint32_t a = (g.ctl & K2_A_ACC) ? acc : s[g.a];
            const uint32_t b = s[g.b];
            const uint32_t r = (g.ctl & K2_XOR) ? (a ^ b ^ g.ma) : ((a ^ g.ma) & (b ^ g.mb));
            if (g.ctl & K2_STORE) s[g.d] = r;
            acc = r;
        }
        out[k] = (acc ^ kp.out_mask) & valid;
    }
}

}  // namespace es
