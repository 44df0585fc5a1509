// es_split.cpp -- split build of the K1 body, for cold (latency-mode) runs.
//
// A one-shot verdict on mult16 spends ~87 % of its time in ptxas compiling
// the one straight-line K1 body, and ptxas time is
// linear in the body (mult8/12/16 at -O1: 59/93/174 ms for 403/782/1,661
// ops).  So the LUT sequence is cut into `parts` phases, each emitted as its
// own PTX module with one device function; the phases compile on parallel
// host threads (es_jit.cpp) and nvJitLink joins them with the skeleton, whose
// body becomes a sequence of calls.
//
// A value defined in one phase and read in a later one passes through a
// per-thread shared-memory slot: stored once after its definition, loaded at
// its first use in every later phase that reads it (slot s of thread t at
// es_slots + (s*threads + t)*4 -- consecutive threads, consecutive banks).
// Cuts are placed where the schedule's crossing count is locally minimal, and
// slots are reused as interval colouring over LUT positions.  PI masks,
// constants and IMAD coefficients are rebuilt inside every phase (FMA pipe).
#include <map>
#include <queue>
#include <sstream>
#include <tuple>
#include <unordered_map>

#include "es_core.h"

namespace es {

bool emit_split_ptx(const LutNet &net, int threads, int parts, const std::string &header,
                    const std::vector<std::string> &outs, const std::string &wlo,
                    const std::string &whi, const std::string &one, SplitPtx *out) {
    const int N = (int)net.is_const.size();
    const int P = net.num_pis;
    const int n = (int)net.luts.size();
    if (parts < 2 || n < parts * 16) return false;
    const bool imad = !one.empty() && getenv("ES_NO_IMAD") == nullptr;
    const bool multi = net.outs.size() > 1 || !net.cof_pis.empty();
    std::vector<int> lut_idx(N, -1);
    for (int i = 0; i < n; ++i) lut_idx[net.luts[i].node] = i;

    // copy c of a multi-output body is folded right after LUT flush_at[c]
    // (-1: before the first LUT), in copy order -- emit_body_ptx's rule
    std::vector<int> flush_at(net.outs.size(), -1);
    if (multi) {
        size_t next = 0;
        auto adv = [&](int pos) {
            while (next < net.outs.size() && (lut_idx[net.outs[next]] < 0 || lut_idx[net.outs[next]] <= pos))
                flush_at[next++] = pos;
        };
        adv(-1);
        for (int i = 0; i < n; ++i) adv(i);
    }
    // last use (LUT position) of every LUT value; the single output is read
    // after the last LUT
    std::vector<int> last_use(n, -1);
    auto leaves_of = [&](const Lut &L, int *ls) {
        int k = 0;
        for (int q = 0; q < L.nleaves; ++q) {
            const int l = L.leaf[q];
            bool seen = false;
            for (int r = 0; r < k; ++r) seen |= ls[r] == l;
            if (!seen) ls[k++] = l;
        }
        return k;
    };
    for (int i = 0; i < n; ++i) {
        int ls[3];
        const int k = leaves_of(net.luts[i], ls);
        for (int q = 0; q < k; ++q)
            if (lut_idx[ls[q]] >= 0) last_use[lut_idx[ls[q]]] = std::max(last_use[lut_idx[ls[q]]], i);
    }
    if (multi) {
        for (size_t c = 0; c < net.outs.size(); ++c)
            if (lut_idx[net.outs[c]] >= 0)
                last_use[lut_idx[net.outs[c]]] = std::max(last_use[lut_idx[net.outs[c]]], flush_at[c]);
    } else if (lut_idx[net.outs[0]] >= 0) {
        last_use[lut_idx[net.outs[0]]] = n;  // read by the return after the last LUT
    }
    // crossing count of a cut before position b: values defined before b and
    // read at or after b
    std::vector<int> cross(n + 2, 0);
    for (int i = 0; i < n; ++i)
        if (last_use[i] > i) { cross[i + 1] += 1; cross[std::min(last_use[i], n) + 1] -= 1; }
    for (int b = 1; b <= n + 1; ++b) cross[b] += cross[b - 1];
    std::vector<int> cuts = {0};
    const int win = std::max(1, n / (parts * 4));  // window 1/2..1/16 of a phase: loads within 8 %
    for (int k = 1; k < parts; ++k) {
        const int target = (int)((int64_t)k * n / parts);
        int best = -1;
        for (int b = std::max(cuts.back() + 8, target - win); b <= std::min(n - 8, target + win); ++b)
            if (best < 0 || cross[b] < cross[best] ||
                (cross[b] == cross[best] && std::abs(b - target) < std::abs(best - target)))
                best = b;
        if (best < 0) return false;
        cuts.push_back(best);
    }
    cuts.push_back(n);
    std::vector<int> phase_of(n + 1, parts - 1);
    for (int ph = 0; ph < parts; ++ph)
        for (int i = cuts[ph]; i < cuts[ph + 1]; ++i) phase_of[i] = ph;
    // slots: values read in a later phase; interval colouring over positions
    // [definition, last use] (a slot is reused by a value defined strictly
    // after the previous owner's last read, so in program order the old
    // value's load precedes the new value's store)
    const int reserved = multi ? 2 : 0;  // the copy fold state (word, copy)
    std::vector<int> slot(n, -1);
    int n_slots = reserved, crossings = 0;
    {
        using Rel = std::pair<int, int>;  // (last use, slot)
        std::priority_queue<Rel, std::vector<Rel>, std::greater<Rel>> busy;
        std::vector<int> free_slots;
        for (int i = 0; i < n; ++i) {
            if (last_use[i] < 0 || phase_of[std::min(last_use[i], n)] == phase_of[i]) continue;
            while (!busy.empty() && busy.top().first < i) { free_slots.push_back(busy.top().second); busy.pop(); }
            int s;
            if (!free_slots.empty()) { s = free_slots.back(); free_slots.pop_back(); }
            else s = n_slots++;
            slot[i] = s;
            busy.push({last_use[i], s});
            ++crossings;
        }
    }
    std::vector<uint8_t> sel(N, 0);
    for (int j = 6; j <= P; ++j) sel[j] = !net.is_const[j];
    for (const Lut &L : net.luts) {
        bool u = true;
        for (int q = 0; q < 3; ++q) u = u && sel[L.leaf[q]];
        sel[L.node] = u;
    }
    auto slot_off = [&](int s) { return (int64_t)s * threads * 4; };

    int total_loads = 0;
    out->phases.clear();
    for (int ph = 0; ph < parts; ++ph) {
        const int a = cuts[ph], b = cuts[ph + 1];
        const bool last = ph == parts - 1;
        std::ostringstream body;
        std::unordered_map<int, std::string> loaded;
        std::unordered_map<uint32_t, int> cidx;
        std::vector<uint32_t> consts;
        std::vector<uint8_t> pi_mask(P + 1, 0), have_bit(N, 0);
        std::map<std::tuple<int, int, int>, std::string> coef;
        auto name = [&](int v) -> std::string {
            const int li = lut_idx[v];
            if (li >= 0) {
                if (phase_of[li] == ph) return "%esq" + std::to_string(li - a);
                auto it = loaded.find(v);
                if (it != loaded.end()) return it->second;
                const std::string r = "%esi" + std::to_string(loaded.size());
                body << "ld.shared.b32 " << r << ", [%esbase+" << slot_off(slot[li]) << "];\n";
                loaded[v] = r;
                return r;
            }
            if (net.is_const[v]) {
                const uint32_t c = net.const_val[v];
                auto it = cidx.find(c);
                int k;
                if (it == cidx.end()) { k = (int)consts.size(); cidx[c] = k; consts.push_back(c); }
                else k = it->second;
                return "%esk" + std::to_string(k);
            }
            pi_mask[v] = 1;
            return "%esm" + std::to_string(v);
        };
        auto bit_of = [&](int u) {
            const std::string bt = "%esb" + std::to_string(u);
            if (!have_bit[u]) {
                have_bit[u] = 1;
                const std::string m = name(u);
                body << "mul.lo.s32 " << bt << ", " << m << ", %esneg1;\n";
            }
            return bt;
        };
        auto coef_reg = [&](int u, int ca, int cb) -> std::string {
            if (ca == cb) return std::to_string(ca);
            auto key = std::make_tuple(u, ca, cb);
            auto it = coef.find(key);
            if (it != coef.end()) return it->second;
            const std::string r = "%esc" + std::to_string(coef.size());
            if (ca == 0 && cb == -1) {
                const std::string m = name(u);
                body << "mov.b32 " << r << ", " << m << ";\n";
            } else if (ca == 0 && cb == 1) {
                const std::string bt = bit_of(u);
                body << "mov.b32 " << r << ", " << bt << ";\n";
            } else {  // mask * (ca - cb) + ca, as emit_body_ptx
                const std::string m = name(u);
                const int f = ca - cb;
                const std::string fr = f == -1 ? "%esneg1" : f == 1 ? "%esone" : f == 2 ? "%escf2" : "%escg2";
                body << "mad.lo.s32 " << r << ", " << m << ", " << fr << ", " << ca << ";\n";
            }
            coef[key] = r;
            return r;
        };
        const std::string o0 = "%eso0", o1 = "%eso1";
        if (multi) {
            if (ph == 0) body << "mov.b32 " << o0 << ", 0;\nmov.b32 " << o1 << ", 0;\n";
            else body << "ld.shared.b32 " << o0 << ", [%esbase];\nld.shared.b32 " << o1 << ", [%esbase+"
                      << slot_off(1) << "];\n";
        }
        size_t next_copy = 0;
        while (next_copy < flush_at.size() && flush_at[next_copy] < a && !(ph == 0 && flush_at[next_copy] == -1))
            ++next_copy;
        auto flush = [&](int pos) {
            while (multi && next_copy < flush_at.size() && flush_at[next_copy] == pos) {
                std::string v = name(net.outs[next_copy]);
                if (net.outs_neg[next_copy]) { body << "not.b32 %est, " << v << ";\n"; v = "%est"; }
                body << "setp.eq.b32 %espz, " << o0 << ", 0;\n"
                     << "selp.b32 " << o0 << ", " << v << ", " << o0 << ", %espz;\n"
                     << "selp.b32 " << o1 << ", " << net.copy_id(next_copy) << ", " << o1 << ", %espz;\n";
                ++next_copy;
            }
        };
        if (ph == 0) flush(-1);
        for (int i = a; i < b; ++i) {
            const Lut &L = net.luts[i];
            const std::string d = "%esq" + std::to_string(i - a);
            ImadPlan pl;
            if (imad && plan_imad(L, sel, &pl)) {
                const std::string S = coef_reg(pl.u, pl.s0, pl.s1), T = coef_reg(pl.u, pl.t0, pl.t1);
                const std::string x = name(pl.x);
                body << "mad.lo.s32 " << d << ", " << x << ", " << S << ", " << T << ";\n";
            } else {
                const std::string l2 = name(L.leaf[2]), l1 = name(L.leaf[1]), l0 = name(L.leaf[0]);
                body << "lop3.b32 " << d << ", " << l2 << ", " << l1 << ", " << l0 << ", " << (int)L.tt << ";\n";
            }
            if (slot[i] >= 0) body << "st.shared.b32 [%esbase+" << slot_off(slot[i]) << "], " << d << ";\n";
            flush(i);
        }
        std::string ret_lo, ret_hi = "0";
        if (last) {
            if (multi) { ret_lo = o0; ret_hi = o1; }
            else {
                ret_lo = name(net.outs[0]);
                if (net.outs_neg[0]) { body << "not.b32 %est, " << ret_lo << ";\n"; ret_lo = "%est"; }
            }
        } else if (multi) {
            body << "st.shared.b32 [%esbase], " << o0 << ";\nst.shared.b32 [%esbase+" << slot_off(1) << "], " << o1
                 << ";\n";
        }
        total_loads += (int)loaded.size();
        std::ostringstream s;
        s << header << "\n.extern .shared .align 16 .b8 es_slots[];\n";
        s << ".visible .func " << (last ? "(.param .b64 es_pr) " : "") << "es_ph_" << ph
          << "(.param .b32 es_pw0, .param .b32 es_pw1, .param .b32 es_pw2)\n{\n";
        s << ".reg .b32 %eswlo, %eswhi, %esone, %esbase, %estmp;\n";
        s << "ld.param.b32 %eswlo, [es_pw0];\nld.param.b32 %eswhi, [es_pw1];\nld.param.b32 %esone, [es_pw2];\n";
        s << "mov.u32 %esbase, %tid.x;\nshl.b32 %esbase, %esbase, 2;\nmov.u32 %estmp, es_slots;\n"
             "add.u32 %esbase, %esbase, %estmp;\n";
        if (b > a) s << ".reg .b32 %esq<" << (b - a) << ">;\n";
        if (!loaded.empty()) s << ".reg .b32 %esi<" << loaded.size() << ">;\n";
        if (!consts.empty()) s << ".reg .b32 %esk<" << consts.size() << ">;\n";
        s << ".reg .b32 %esm<" << (P + 1) << ">;\n.reg .b32 %esb<" << N << ">;\n";
        if (!coef.empty()) s << ".reg .b32 %esc<" << coef.size() << ">;\n";
        s << ".reg .b32 %est, %eso0, %eso1;\n.reg .pred %espz;\n.reg .b64 %esr;\n";
        for (size_t k = 0; k < consts.size(); ++k) s << "mov.b32 %esk" << k << ", " << consts[k] << ";\n";
        if (imad)
            s << ".reg .b32 %esneg1, %escf2, %escg2;\nneg.s32 %esneg1, %esone;\nadd.s32 %escf2, %esone, %esone;\n"
                 "neg.s32 %escg2, %escf2;\n";
        for (int j = 6; j <= P; ++j) {
            if (!pi_mask[j]) continue;
            const int bit = net.pi_bit[j];
            const std::string src = bit < 32 ? "%eswlo" : "%eswhi";
            if (imad) {
                s << "mul.lo.u32 %esm" << j << ", " << src << ", " << (1u << (31 - (bit & 31))) << ";\n";
                s << "mul.hi.s32 %esm" << j << ", %esm" << j << ", %esone;\n";
            } else {
                s << "shl.b32 %esm" << j << ", " << src << ", " << (31 - (bit & 31)) << ";\n";
                s << "shr.s32 %esm" << j << ", %esm" << j << ", 31;\n";
            }
        }
        s << body.str();
        if (last) s << "mov.b64 %esr, {" << ret_lo << ", " << ret_hi << "};\nst.param.b64 [es_pr], %esr;\n";
        s << "ret;\n}\n";
        out->phases.push_back(s.str());
    }
    // the caller: module-scope declarations and the call sequence
    std::ostringstream dc, cb;
    for (int ph = 0; ph < parts; ++ph)
        dc << ".extern .func " << (ph == parts - 1 ? "(.param .b64 es_pr) " : "") << "es_ph_" << ph
           << "(.param .b32 es_pw0, .param .b32 es_pw1, .param .b32 es_pw2);\n";
    cb << "{\n.reg .b64 %esret;\n";
    for (int ph = 0; ph < parts; ++ph) {
        const bool last = ph == parts - 1;
        cb << "{\n.param .b32 es_a0;\n.param .b32 es_a1;\n.param .b32 es_a2;\n";
        if (last) cb << ".param .b64 es_r;\n";
        cb << "st.param.b32 [es_a0], " << wlo << ";\nst.param.b32 [es_a1], " << whi << ";\nst.param.b32 [es_a2], "
           << one << ";\n";
        cb << "call.uni " << (last ? "(es_r), " : "") << "es_ph_" << ph << ", (es_a0, es_a1, es_a2);\n";
        if (last) cb << "ld.param.b64 %esret, [es_r];\n";
        cb << "}\n";
    }
    if (multi) cb << "mov.b64 {" << outs[0] << ", " << outs[1] << "}, %esret;\n";
    else cb << "cvt.u32.u64 " << outs[0] << ", %esret;\n";
    cb << "}\n";
    out->decls = dc.str();
    out->call_body = cb.str();
    out->slots = n_slots;
    out->crossings = crossings;
    out->loads = total_loads;
    out->cuts.assign(cuts.begin(), cuts.end() - 1);
    return true;
}

}  // namespace es
