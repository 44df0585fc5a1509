// es_spill.cpp -- shared-memory overflow slots for the K1 body (north_star (2):
// "slots in shared memory, overflow spilled with coalesced stores").
//
// K1 keeps every LUT value in a register.  At 255 registers a CTA of 256
// threads leaves 8 warps per SM (2 per scheduler), and the deepest cofactor
// variants do not fit at all (mult16 with 5 cofactor PIs: 446 live values;
// ptxas spills to local memory and the kernel runs 2x slower).  This pass
// rewrites the straight-line body so that at most `budget` values are live in
// registers at any point of the schedule: when the live set would exceed it,
// the value whose next use lies farthest ahead (Belady's rule, optimal for a
// straight-line schedule) moves to a per-thread shared-memory slot -- stored
// once, at its first eviction, and reloaded before each later use that finds
// it evicted.  Slot s of thread t sits at es_slots + (s * threads + t) * 4, so
// a warp's access is 32 consecutive words: one wavefront, no bank conflicts.
// Slots are reused by interval colouring over [store, last reload].
//
// The loads and stores run on the LSU/MIO path, which K1 otherwise leaves
// idle, while the ALU pipe keeps the LOP3s; the freed registers buy either
// more resident warps (a 168-register cap gives 12 warps per SM instead of
// 8) or a deeper cofactor variant without local-memory spills.
#include <algorithm>
#include <map>
#include <queue>
#include <set>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "es_core.h"

namespace es {

namespace {

struct Ins {
    std::string op;
    std::vector<std::string> opnd;  // operand text, [0] = destination
    std::string raw;                // the original line (non-instructions)
    bool is_ins = false;
};

// a spillable value: a single-definition %es register (the emitter's LUT,
// PI-mask, bit and coefficient registers); constants, the -1 register, the
// output-fold temporaries and predicates stay in registers
bool spillable(const std::string &r) {
    if (r.size() < 4 || r.compare(0, 3, "%es") != 0) return false;
    if (r == "%espz" || r == "%est" || r == "%esneg1") return false;
    const char c = r[3];
    return c == 'q' || c == 'm' || c == 'b' || c == 'c' || c == 'p';
}

bool parse(const std::string &line, Ins *out) {
    out->raw = line;
    size_t a = line.find_first_not_of(" \t");
    if (a == std::string::npos || line[a] == '.' || line[a] == '{' || line[a] == '}' || line[a] == '/')
        return false;
    const size_t sp = line.find_first_of(" \t", a);
    const size_t semi = line.rfind(';');
    if (sp == std::string::npos || semi == std::string::npos) return false;
    out->op = line.substr(a, sp - a);
    std::string rest = line.substr(sp + 1, semi - sp - 1);
    std::stringstream ss(rest);
    for (std::string t; std::getline(ss, t, ',');) {
        const size_t b = t.find_first_not_of(" \t"), e = t.find_last_not_of(" \t");
        out->opnd.push_back(b == std::string::npos ? "" : t.substr(b, e - b + 1));
    }
    out->is_ins = !out->opnd.empty();
    return out->is_ins;
}

}  // namespace

std::string spill_body(const std::string &body, int budget, int threads, SpillStats *st) {
    std::vector<Ins> prog;
    {
        std::stringstream in(body);
        for (std::string line; std::getline(in, line);) {
            Ins x;
            parse(line, &x);
            prog.push_back(std::move(x));
        }
    }
    const int n = (int)prog.size();
    // values: definition index and use positions
    std::unordered_map<std::string, int> id;
    std::vector<std::string> name;
    std::vector<int> def;
    std::vector<std::vector<int>> uses;
    auto vid = [&](const std::string &r) {
        auto it = id.find(r);
        if (it != id.end()) return it->second;
        const int k = (int)name.size();
        id[r] = k;
        name.push_back(r);
        def.push_back(-1);
        uses.emplace_back();
        return k;
    };
    std::vector<std::vector<int>> srcs(n);
    std::vector<int> dst(n, -1);
    for (int i = 0; i < n; ++i) {
        const Ins &x = prog[i];
        if (!x.is_ins) continue;
        for (size_t q = 1; q < x.opnd.size(); ++q)
            if (spillable(x.opnd[q])) {
                const int v = vid(x.opnd[q]);
                if (std::find(srcs[i].begin(), srcs[i].end(), v) == srcs[i].end()) srcs[i].push_back(v);
            }
        // st.* has no destination; everything else the emitter writes does
        if (x.op.compare(0, 3, "st.") != 0 && spillable(x.opnd[0])) {
            const int v = vid(x.opnd[0]);
            if (def[v] >= 0) return body;  // not single-definition: leave the body alone
            def[v] = i;
            dst[i] = v;
        }
    }
    const int V = (int)name.size();
    for (int i = 0; i < n; ++i)
        for (int v : srcs[i]) uses[v].push_back(i);
    for (int v = 0; v < V; ++v)
        if (def[v] < 0 && !uses[v].empty()) return body;  // read but never defined here

    // pass 1: Belady over the schedule
    std::vector<size_t> ptr(V, 0);
    auto next_use = [&](int v, int after) -> int {  // first use > after, or INT_MAX
        size_t &p = ptr[v];
        while (p < uses[v].size() && uses[v][p] <= after) ++p;
        return p < uses[v].size() ? uses[v][p] : 1 << 30;
    };
    std::set<std::pair<int, int>> res;  // (next use, value) of the register-resident values
    std::vector<int> key(V, -1);        // value's key in res (-1: not resident)
    std::vector<uint8_t> in_mem(V, 0), store(V, 0);
    std::vector<std::vector<int>> reload(n);  // values reloaded before instruction i
    // a value is stored when it is first evicted (it is still in its register
    // there): before instruction i (evicted to make room for i's reloads) or
    // after it (evicted for i's result)
    std::vector<std::vector<int>> store_pre(n), store_post(n);
    std::vector<int> store_at(V, -1), last_reload(V, -1);
    int pos = 0;
    bool post = false;
    auto evict_to = [&](int cap, const std::vector<int> &keep) {
        while ((int)res.size() > cap) {
            auto it = std::prev(res.end());
            while (std::find(keep.begin(), keep.end(), it->second) != keep.end()) {
                if (it == res.begin()) return;
                it = std::prev(it);
            }
            const int v = it->second;
            res.erase(it);
            key[v] = -1;
            if (!in_mem[v]) {
                in_mem[v] = 1;
                store[v] = 1;
                store_at[v] = pos;
                (post ? store_post : store_pre)[pos].push_back(v);
            }
        }
    };
    int peak = 0;
    for (int i = 0; i < n; ++i) {
        if (!prog[i].is_ins) continue;
        pos = i;
        post = false;
        for (int v : srcs[i])
            if (key[v] < 0) {
                reload[i].push_back(v);
                last_reload[v] = i;
                key[v] = i;
                res.insert({i, v});
            }
        evict_to(budget, srcs[i]);
        peak = std::max(peak, (int)res.size());
        for (int v : srcs[i]) {
            res.erase({key[v], v});
            const int nu = next_use(v, i);
            if (nu >= (1 << 30)) { key[v] = -1; continue; }
            key[v] = nu;
            res.insert({nu, v});
        }
        if (dst[i] >= 0) {
            const int v = dst[i];
            const int nu = next_use(v, i);
            if (nu < (1 << 30)) {
                key[v] = nu;
                res.insert({nu, v});
                post = true;
                evict_to(budget, {});
            }
        }
    }
    // slots: interval colouring of the stored values over [store, last reload]
    // (a slot whose last reload is at instruction i is free only after i: a
    // store emitted at i may precede i's reloads)
    std::vector<int> slot(V, -1), order;
    for (int v = 0; v < V; ++v)
        if (store[v]) order.push_back(v);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return store_at[a] < store_at[b]; });
    int n_slots = 0;
    {
        using Rel = std::pair<int, int>;  // (last use, slot)
        std::priority_queue<Rel, std::vector<Rel>, std::greater<Rel>> busy;
        std::vector<int> free_slots;
        for (int v : order) {
            while (!busy.empty() && busy.top().first < store_at[v]) { free_slots.push_back(busy.top().second); busy.pop(); }
            int s;
            if (!free_slots.empty()) { s = free_slots.back(); free_slots.pop_back(); }
            else s = n_slots++;
            slot[v] = s;
            busy.push({std::max(last_reload[v], store_at[v]), s});
        }
    }
    if (n_slots == 0) {
        if (st) *st = SpillStats{0, 0, 0, peak};
        return body;
    }
    // pass 2: emit with the stores after definitions and the reloads renamed
    std::vector<std::string> cur(V);
    for (int v = 0; v < V; ++v) cur[v] = name[v];
    int n_loads = 0, n_stores = 0;
    std::ostringstream o;
    bool decl_done = false;
    auto addr = [&](int v) { return "[%esbase+" + std::to_string((long long)slot[v] * threads * 4) + "]"; };
    for (int i = 0; i < n; ++i) {
        const Ins &x = prog[i];
        if (!x.is_ins) {
            o << x.raw << "\n";
            if (!decl_done && x.raw.find('{') != std::string::npos) {
                o << ".reg .b32 %esbase, %esbtmp;\n.reg .b32 %esr<@NR@>;\n"
                  << "mov.u32 %esbase, %tid.x;\nshl.b32 %esbase, %esbase, 2;\n"
                  << "mov.u32 %esbtmp, es_slots;\nadd.u32 %esbase, %esbase, %esbtmp;\n";
                decl_done = true;
            }
            continue;
        }
        for (int v : store_pre[i]) {
            o << "st.shared.b32 " << addr(v) << ", " << cur[v] << ";\n";
            ++n_stores;
        }
        for (int v : reload[i]) {
            cur[v] = "%esr" + std::to_string(n_loads++);
            o << "ld.shared.b32 " << cur[v] << ", " << addr(v) << ";\n";
        }
        o << x.op << " ";
        for (size_t q = 0; q < x.opnd.size(); ++q) {
            const std::string &r = x.opnd[q];
            std::string t = r;
            if (q > 0 && spillable(r)) t = cur[id[r]];
            o << (q ? ", " : "") << t;
        }
        o << ";\n";
        for (int v : store_post[i]) {
            o << "st.shared.b32 " << addr(v) << ", " << cur[v] << ";\n";
            ++n_stores;
        }
    }
    std::string out = o.str();
    const size_t at = out.find("@NR@");
    if (at != std::string::npos) out.replace(at, 4, std::to_string(std::max(1, n_loads)));
    if (st) *st = SpillStats{n_slots, n_loads, n_stores, peak};
    return out;
}

}  // namespace es
