// es_aiger.cpp -- AIGER ingest and XOR recovery in C++ (SURVEY 8(f) next-4).
//
//  parse_aiger : cecprove/aiger.py:44-194 -- ASCII ("aag") and binary ("aig")
//                combinational files, the same header checks (:29-41), the
//                same out-of-order-definition DFS (:63-92, identical emission
//                order, so gate numbering matches), the same errors
//                (MalformedHeader / LatchesUnsupported / DanglingLiteral /
//                cyclic definitions) as return codes;
//  detect_xors : cecprove/transform.py:79-119 -- AND(~n1, ~n2) with
//                n1 = AND(u, v), n2 = AND(~u, ~v) folds to u XOR v, then the
//                reachable rebuild (transform.py:31-60, keep_all_pis);
//  write_aiger : cecprove/aiger.py:197-225 -- ASCII, XOR as three ANDs.
// Every circuit goes through the reference's builder (es_xag.h), so the
// result is gate-for-gate the reference's Xag: the ES engine then compiles
// the same program (same G) the reference would.
#include <algorithm>
#include <array>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/es_b200.h"
#include "es_xag.h"

namespace es {

void set_error(const std::string &m);


namespace {

struct AigErr {
    int code;
    std::string msg;
};

XagC finish(const Builder &b, const std::vector<Lit> &outs) {
    XagC x;
    x.num_pis = b.num_pis;
    x.kind = b.kind;
    x.in0 = b.in0;
    x.in1 = b.in1;
    for (const Lit &l : outs) x.outs.push_back(l.pack());
    return x;
}

// split on ASCII whitespace (bytes.split())
std::vector<std::string> split_ws(const std::string &s) {
    std::vector<std::string> out;
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && isspace((unsigned char)s[i])) ++i;
        size_t j = i;
        while (j < s.size() && !isspace((unsigned char)s[j])) ++j;
        if (j > i) out.push_back(s.substr(i, j - i));
        i = j;
    }
    return out;
}

bool parse_int(const std::string &t, long long *v) {  // Python int() on a token
    if (t.empty()) return false;
    size_t i = 0;
    bool neg = false;
    if (t[0] == '+' || t[0] == '-') { neg = t[0] == '-'; i = 1; }
    if (i >= t.size()) return false;
    long long r = 0;
    for (; i < t.size(); ++i) {
        if (t[i] == '_' && i + 1 < t.size() && i > 0 && isdigit((unsigned char)t[i - 1])) continue;
        if (!isdigit((unsigned char)t[i])) return false;
        r = r * 10 + (t[i] - '0');
        if (r > (1ll << 40)) return false;
    }
    *v = neg ? -r : r;
    return true;
}

XagC build(int num_in, long long m, int num_and, const std::vector<long long> &def_order,
           const std::unordered_map<long long, std::pair<long long, long long>> &and_defs,
           const std::vector<long long> &out_lits) {
    if ((int)and_defs.size() != num_and) throw AigErr{ES_E_AIGER_HEADER, "duplicate or missing AND definitions"};
    Builder b(num_in);
    std::unordered_map<long long, Lit> lit_of;
    lit_of[0] = kFalse;
    std::unordered_map<long long, int> state;  // 1 on stack, 2 emitted
    std::vector<long long> order;
    auto st_of = [&](long long v) { auto it = state.find(v); return it == state.end() ? 0 : it->second; };
    for (long long root : def_order) {
        if (st_of(root) == 2) continue;
        std::vector<std::pair<long long, bool>> stack{{root, false}};
        while (!stack.empty()) {
            auto [v, expanded] = stack.back();
            stack.pop_back();
            if (expanded) { state[v] = 2; order.push_back(v); continue; }
            if (st_of(v) == 2) continue;
            if (st_of(v) == 1) throw AigErr{ES_E_AIGER, "cyclic AND definitions"};
            state[v] = 1;
            stack.push_back({v, true});
            const auto &d = and_defs.at(v);
            for (long long dl : {d.first, d.second}) {
                const long long dv = dl >> 1;
                if (dv == 0 || (1 <= dv && dv <= num_in) || st_of(dv) == 2) continue;
                if (!and_defs.count(dv)) throw AigErr{ES_E_AIGER_DANGLING, "variable " + std::to_string(dv) + " is never defined"};
                if (st_of(dv) == 1) throw AigErr{ES_E_AIGER, "cyclic AND definitions"};
                stack.push_back({dv, false});
            }
        }
    }
    auto lit = [&](long long al) -> Lit {
        const long long var = al >> 1;
        const bool neg = al & 1;
        if (var > m) throw AigErr{ES_E_AIGER_DANGLING, "literal " + std::to_string(al) + " exceeds declared maximum"};
        if (1 <= var && var <= num_in) return Lit{(int32_t)var, neg};
        auto it = lit_of.find(var);
        if (it == lit_of.end()) throw AigErr{ES_E_AIGER_DANGLING, "literal " + std::to_string(al) + " undefined"};
        return Lit{it->second.node, it->second.neg != neg};
    };
    for (long long v : order) {
        const auto &d = and_defs.at(v);
        lit_of[v] = b.add_and(lit(d.first), lit(d.second));
    }
    std::vector<Lit> outs;
    for (long long ol : out_lits) {
        const long long var = ol >> 1;
        if (var > m || (var > num_in && !lit_of.count(var) && var != 0))
            throw AigErr{ES_E_AIGER_DANGLING, "output literal " + std::to_string(ol) + " undefined"};
        outs.push_back(lit(ol));
    }
    return finish(b, outs);
}

XagC parse(const uint8_t *data, size_t len) {
    const char *p = (const char *)data;
    const void *nl = memchr(p, '\n', len);
    if (!nl) throw AigErr{ES_E_AIGER_HEADER, "missing header line"};
    const size_t hl = (const char *)nl - p;
    const std::vector<std::string> parts = split_ws(std::string(p, hl));
    if (parts.size() < 6 || (parts[0] != "aag" && parts[0] != "aig"))
        throw AigErr{ES_E_AIGER_HEADER, "bad AIGER header"};
    long long f[5];
    for (int k = 0; k < 5; ++k)
        if (!parse_int(parts[1 + k], &f[k])) throw AigErr{ES_E_AIGER_HEADER, "non-integer header field"};
    for (size_t k = 6; k < parts.size(); ++k) {
        long long v;
        if (!parse_int(parts[k], &v) || v != 0)
            throw AigErr{ES_E_AIGER_HEADER, "extension sections (B/C/J/F) are not supported"};
    }
    const long long m = f[0], ni = f[1], nl2 = f[2], no = f[3], na = f[4];
    if (m < ni + nl2 + na) throw AigErr{ES_E_AIGER_HEADER, "declared maximum below I+L+A"};
    if (nl2) throw AigErr{ES_E_AIGER_LATCHES, std::to_string(nl2) + " latches declared"};
    if (ni < 0 || no < 0 || na < 0 || ni > (1 << 26) || na > (1 << 28) || no > (1 << 26))
        throw AigErr{ES_E_AIGER_HEADER, "header sizes out of range"};
    const char *body = p + hl + 1;
    const size_t blen = len - hl - 1;
    std::unordered_map<long long, std::pair<long long, long long>> and_defs;
    std::vector<long long> def_order, out_lits;
    if (parts[0] == "aag") {
        const long long need = ni + no + na;
        std::vector<std::vector<long long>> fields;
        size_t i = 0;
        while (i <= blen && (long long)fields.size() < need) {
            size_t j = i;
            while (j < blen && body[j] != '\n') ++j;
            const std::vector<std::string> toks = split_ws(std::string(body + i, j - i));
            if (!toks.empty()) {
                std::vector<long long> row;
                for (const auto &t : toks) {
                    long long v;
                    if (!parse_int(t, &v)) throw AigErr{ES_E_AIGER_HEADER, "non-numeric body line"};
                    row.push_back(v);
                }
                fields.push_back(row);
            }
            i = j + 1;
        }
        if ((long long)fields.size() < need) throw AigErr{ES_E_AIGER_HEADER, "truncated file body"};
        size_t pos = 0;
        for (long long k = 0; k < ni; ++k) {
            const auto &row = fields[pos + k];
            if (row.size() != 1 || (row[0] & 1) || row[0] == 0) throw AigErr{ES_E_AIGER_HEADER, "bad input literal line"};
        }
        pos += ni;
        for (long long k = 0; k < no; ++k) {
            const auto &row = fields[pos + k];
            if (row.size() != 1) throw AigErr{ES_E_AIGER_HEADER, "bad output literal line"};
            out_lits.push_back(row[0]);
        }
        pos += no;
        for (long long k = 0; k < na; ++k) {
            const auto &row = fields[pos + k];
            if (row.size() != 3 || (row[0] & 1)) throw AigErr{ES_E_AIGER_HEADER, "bad AND line"};
            const long long var = row[0] >> 1;
            if (var <= ni || var > m || and_defs.count(var)) throw AigErr{ES_E_AIGER_HEADER, "AND defines illegal variable"};
            and_defs[var] = {row[1], row[2]};
            def_order.push_back(var);
        }
    } else {
        size_t pos = 0;
        for (long long k = 0; k < no; ++k) {
            const void *e = memchr(body + pos, '\n', blen - pos);
            if (!e) throw AigErr{ES_E_AIGER_HEADER, "truncated output section"};
            const size_t end = (const char *)e - body;
            // int() tolerates surrounding whitespace
            std::vector<std::string> t = split_ws(std::string(body + pos, end - pos));
            long long v;
            if (t.size() != 1 || !parse_int(t[0], &v)) throw AigErr{ES_E_AIGER_HEADER, "bad output literal"};
            out_lits.push_back(v);
            pos = end + 1;
        }
        auto delta = [&]() -> long long {
            long long value = 0;
            int shift = 0;
            for (;;) {
                if (pos >= blen) throw AigErr{ES_E_AIGER_HEADER, "truncated binary AND section"};
                const unsigned char byte = (unsigned char)body[pos++];
                if (shift < 62) value |= (long long)(byte & 0x7F) << shift;
                if (!(byte & 0x80)) return value;
                shift += 7;
            }
        };
        for (long long k = 0; k < na; ++k) {
            const long long lhs = 2 * (ni + k + 1);
            const long long d0 = delta(), d1 = delta();
            const long long r0 = lhs - d0, r1 = r0 - d1;
            if (r0 < 0 || r1 < 0) throw AigErr{ES_E_AIGER_DANGLING, "binary AND decodes to negative fanin"};
            and_defs[lhs >> 1] = {r0, r1};
            def_order.push_back(lhs >> 1);
        }
    }
    return build((int)ni, m, (int)na, def_order, and_defs, out_lits);
}

// transform.py:31-60 with keep_all_pis: rebuild what the outputs reach
XagC rebuild(const XagC &x) {
    const int P = x.num_pis, FG = 1 + P, NN = FG + (int)x.kind.size();
    std::vector<uint8_t> alive(NN, 0);
    alive[0] = 1;
    std::vector<int> st;
    for (uint32_t o : x.outs) st.push_back((int)(o >> 1));
    while (!st.empty()) {
        const int n = st.back();
        st.pop_back();
        if (alive[n]) continue;
        alive[n] = 1;
        if (n >= FG) { st.push_back((int)(x.in0[n - FG] >> 1)); st.push_back((int)(x.in1[n - FG] >> 1)); }
    }
    Builder b(P);
    std::vector<Lit> lit_of(NN, kFalse);
    for (int i = 1; i <= P; ++i) lit_of[i] = Lit{i, false};
    auto remap = [&](uint32_t l) { const Lit &bl = lit_of[l >> 1]; return Lit{bl.node, bl.neg != (bool)(l & 1)}; };
    for (int g = 0; g < (int)x.kind.size(); ++g) {
        if (!alive[FG + g]) continue;
        lit_of[FG + g] = x.kind[g] ? b.add_xor(remap(x.in0[g]), remap(x.in1[g]))
                                   : b.add_and(remap(x.in0[g]), remap(x.in1[g]));
    }
    std::vector<Lit> outs;
    for (uint32_t o : x.outs) outs.push_back(remap(o));
    return finish(b, outs);
}

XagC detect_xors(const XagC &x) {  // transform.py:79-119
    const int P = x.num_pis, FG = 1 + P, NN = FG + (int)x.kind.size();
    Builder b(P);
    std::vector<Lit> lit_of(NN, kFalse);
    for (int i = 1; i <= P; ++i) lit_of[i] = Lit{i, false};
    auto remap = [&](uint32_t l) { const Lit &bl = lit_of[l >> 1]; return Lit{bl.node, bl.neg != (bool)(l & 1)}; };
    auto and_fanins = [&](int node, uint32_t *f0, uint32_t *f1) {
        if (node < FG) return false;  // PI or constant
        if (x.kind[node - FG] != 0) return false;
        *f0 = x.in0[node - FG];
        *f1 = x.in1[node - FG];
        return true;
    };
    for (int g = 0; g < (int)x.kind.size(); ++g) {
        bool folded = false;
        Lit res = kFalse;
        if (x.kind[g] == 0 && (x.in0[g] & 1) && (x.in1[g] & 1)) {
            uint32_t a0, a1, b0, b1;
            if (and_fanins((int)(x.in0[g] >> 1), &a0, &a1) && and_fanins((int)(x.in1[g] >> 1), &b0, &b1)) {
                // {f2 packs} == {~f1[0], ~f1[1]} as sets
                const uint32_t n0 = a0 ^ 1u, n1 = a1 ^ 1u;
                std::unordered_set<uint32_t> s2{b0, b1}, s1{n0, n1};
                if (s1 == s2) { res = b.add_xor(remap(a0), remap(a1)); folded = true; }
            }
        }
        if (!folded)
            res = x.kind[g] ? b.add_xor(remap(x.in0[g]), remap(x.in1[g])) : b.add_and(remap(x.in0[g]), remap(x.in1[g]));
        lit_of[FG + g] = res;
    }
    std::vector<Lit> outs;
    for (uint32_t o : x.outs) outs.push_back(remap(o));
    return rebuild(finish(b, outs));
}

std::string write_aiger(const XagC &x) {  // aiger.py:197-225
    const int ni = x.num_pis, FG = 1 + ni;
    std::vector<std::array<uint32_t, 3>> ands;
    std::vector<uint32_t> lit_of(FG + x.kind.size(), 0);
    for (int i = 1; i <= ni; ++i) lit_of[i] = 2u * i;
    auto fresh = [&](uint32_t r0, uint32_t r1) {
        const uint32_t lhs = 2u * (uint32_t)(ni + ands.size() + 1);
        ands.push_back({lhs, std::max(r0, r1), std::min(r0, r1)});
        return lhs;
    };
    for (size_t g = 0; g < x.kind.size(); ++g) {
        const uint32_t a = lit_of[x.in0[g] >> 1] ^ (x.in0[g] & 1), b = lit_of[x.in1[g] >> 1] ^ (x.in1[g] & 1);
        if (x.kind[g] == 0) lit_of[FG + g] = fresh(a, b);
        else {
            const uint32_t n1 = fresh(a, b ^ 1u), n2 = fresh(a ^ 1u, b);
            lit_of[FG + g] = fresh(n1 ^ 1u, n2 ^ 1u) ^ 1u;
        }
    }
    std::string s = "aag " + std::to_string(ni + ands.size()) + " " + std::to_string(ni) + " 0 " +
                    std::to_string(x.outs.size()) + " " + std::to_string(ands.size());
    for (int i = 1; i <= ni; ++i) s += "\n" + std::to_string(2 * i);
    for (uint32_t o : x.outs) s += "\n" + std::to_string(lit_of[o >> 1] ^ (o & 1));
    for (const auto &a : ands) s += "\n" + std::to_string(a[0]) + " " + std::to_string(a[1]) + " " + std::to_string(a[2]);
    return s + "\n";
}

XagC from_arrays(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                 const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits) {
    XagC x;
    x.num_pis = num_pis;
    x.kind.assign(kind, kind + num_gates);
    x.in0.assign(in0, in0 + num_gates);
    x.in1.assign(in1, in1 + num_gates);
    x.outs.assign(out_lits, out_lits + num_outputs);
    const int FG = 1 + num_pis;
    for (int g = 0; g < num_gates; ++g)
        if ((int)(in0[g] >> 1) >= FG + g || (int)(in1[g] >> 1) >= FG + g) throw AigErr{ES_E_BAD_PROGRAM, "XAG not topological"};
    for (int o = 0; o < num_outputs; ++o)
        if ((int)(out_lits[o] >> 1) >= FG + num_gates) throw AigErr{ES_E_BAD_PROGRAM, "output references unknown node"};
    return x;
}

}  // namespace

int aiger_parse(const uint8_t *data, int64_t len, int32_t xors, XagC **out) {
    try {
        XagC x = parse(data, (size_t)len);
        *out = new XagC(xors ? detect_xors(x) : std::move(x));
        return ES_OK;
    } catch (const AigErr &e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception &e) {
        set_error(std::string("AIGER: ") + e.what());
        return ES_E_AIGER;
    }
}

int xag_detect_xors(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits, XagC **out) {
    try {
        *out = new XagC(detect_xors(from_arrays(num_pis, num_gates, kind, in0, in1, num_outputs, out_lits)));
        return ES_OK;
    } catch (const AigErr &e) {
        set_error(e.msg);
        return e.code;
    }
}

int64_t aiger_write(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits, char *buf,
                    int64_t cap) {
    try {
        const std::string s = write_aiger(from_arrays(num_pis, num_gates, kind, in0, in1, num_outputs, out_lits));
        if (buf && cap > 0) {
            const int64_t n = std::min<int64_t>(cap, (int64_t)s.size());
            std::memcpy(buf, s.data(), (size_t)n);
        }
        return (int64_t)s.size();
    } catch (const AigErr &e) {
        set_error(e.msg);
        return e.code;
    }
}

}  // namespace es
