// es_abi.cpp -- extern "C" entry points declared in include/es_b200.h.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>
#include <string>
#include <vector>

#include "es_core.h"
#include "es_extract.h"
#include "es_jit.h"
#include "es_k2prog.h"
#include "es_xag.h"

namespace es {

thread_local std::string t_err;
void set_error(const std::string &m) { t_err = m; }

int run_one(const es_prog *prog, const es_run_opts *opts, es_result *out);
int run_batch_jit(int n_jobs, const es_prog *progs, const es_run_opts *opts, es_result *outs);
void k4_prebuild(int n, const es_prog *progs, const K2Prog *const *kps);
int run_batch(int n_jobs, const es_prog *progs, const es_run_opts *opts, es_result *outs,
              const K2Prog *const *prebuilt = nullptr);
int session_open(const es_prog *prog, const es_run_opts *opts, void **out);
int session_geometry(const void *s, uint64_t *n_chunks, uint64_t *ppc, int32_t *luts, int32_t *regs);
int session_launch(void *s, void *stream, uint64_t *best_dev, uint64_t chunk_begin,
                   uint64_t chunk_end, int rank, int world);
void session_close(void *s);
void runtime_shutdown();
int alu_peak(int dev, double *lane_ops_per_s, double *ms_out);
int fma_peak(int dev, double *lane_ops_per_s, double *ms_out);
int smem_peak(int dev, double *bytes_per_s, double *ms_out);
int ipc_alloc(int dev, void **ptr, unsigned char *handle);
int ipc_open(int dev, const unsigned char *handle, void **ptr);
int ipc_close(int dev, void *ptr, int owner);
int word_io(int dev, void *ptr, uint64_t *value, int write);
int peer_arm(void *stream, void *word);
int peer_arrive_wait(void *stream, void *word, int world, void *out);
int sim_run(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
            const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
            uint64_t *node_words, double *device_ms);
int sim_ones(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
             const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
             int64_t *ones, double *device_ms);
int sim_run_device(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                   const uint32_t *in1, const uint64_t *d_pi_words, int64_t words, void *stream,
                   uint64_t *d_node_words, void **prog_cache);
void sim_prog_free(void *prog_cache);
int aiger_parse(const uint8_t *data, int64_t len, int32_t xors, XagC **out);
int xag_detect_xors(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits, XagC **out);
int64_t aiger_write(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits, char *buf,
                    int64_t cap);
int sim_levels(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
              const uint32_t *in1);
int sim_classes(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
                int32_t *class_id, uint8_t *polarity, int32_t *n_classes, double *device_ms);

// k = cofactor PIs (0: none), chosen as the runtime does (rank_cofactor_pis)
static int map_prog(const es_prog *prog, LutNet *net, int k = 0, int copies = 0) {
    if (!prog || prog->num_instrs < 1) { set_error("empty program"); return ES_E_BAD_PROGRAM; }
    if (k < 0 || k > kMaxCofactorPis) { set_error("cofactor PIs must be 0.." + std::to_string(kMaxCofactorPis)); return ES_E_BAD_ARG; }
    Dag dag;
    std::string err;
    int rc = build_dag(*prog, &dag, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    if (k == 0) { map_luts(dag, net); return ES_OK; }
    std::vector<int32_t> pis = rank_cofactor_pis(dag, k);
    std::sort(pis.begin(), pis.end());
    if ((int)pis.size() != k) { set_error("fewer word PIs than cofactor PIs"); return ES_E_BAD_ARG; }
    if (copies < 0 || copies > (1 << k)) { set_error("copies must be 0..2^k"); return ES_E_BAD_ARG; }
    std::vector<int32_t> ids;
    for (int c = 0; c < copies; ++c) ids.push_back(c);
    map_cofactored(dag, pis, net, copies && copies < (1 << k) ? &ids : nullptr);
    return ES_OK;
}

struct Batch {
    std::vector<SubMiterC> subs;
};

}  // namespace es

using namespace es;

extern "C" {

int32_t es_compile(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                   const uint32_t *in1, uint32_t out_lit, int8_t *op, int32_t *dst, int32_t *src0,
                   uint8_t *neg0, int32_t *src1, uint8_t *neg1, int32_t *pi,
                   int32_t *num_registers) {
    int32_t rc = ref_compile(num_pis, num_gates, kind, in0, in1, out_lit, op, dst, src0, neg0,
                             src1, neg1, pi, num_registers);
    if (rc == ES_E_TOO_MANY_INPUTS) set_error(std::to_string(num_pis) + " PIs exceeds the 40 ceiling");
    else if (rc < 0) set_error("malformed XAG");
    return rc;
}

int32_t es_run(const es_prog *prog, const es_run_opts *opts, es_result *out) {
    if (!prog || !out) { set_error("null argument"); return ES_E_BAD_ARG; }
    return run_one(prog, opts, out);
}

int32_t es_device_count(int32_t *n) {
    if (!n) { set_error("null argument"); return ES_E_BAD_ARG; }
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) { cudaGetLastError(); c = 0; }
    *n = c;
    return ES_OK;
}

int32_t es_run_batch(int32_t n_jobs, const es_prog *progs, const es_run_opts *opts,
                     es_result *outs) {
    if (n_jobs < 0 || (n_jobs > 0 && (!progs || !outs))) { set_error("bad batch"); return ES_E_BAD_ARG; }
    return run_batch(n_jobs, progs, opts, outs);
}

int32_t es_session_open(const es_prog *prog, const es_run_opts *opts, es_session **out) {
    void *s = nullptr;
    int rc = session_open(prog, opts, &s);
    *out = (es_session *)s;
    return rc;
}

int32_t es_session_geometry(const es_session *s, uint64_t *n_chunks, uint64_t *ppc,
                            int32_t *num_luts, int32_t *regs) {
    if (!s) return ES_E_BAD_ARG;
    return session_geometry(s, n_chunks, ppc, num_luts, regs);
}

int32_t es_session_launch(es_session *s, void *stream, uint64_t *best_dev, uint64_t chunk_begin,
                          uint64_t chunk_end, int32_t rank, int32_t world) {
    if (!s || !best_dev) { set_error("null argument"); return ES_E_BAD_ARG; }
    return session_launch(s, stream, best_dev, chunk_begin, chunk_end, rank, world);
}

void es_session_close(es_session *s) { session_close(s); }

int32_t es_map_stats(const es_prog *prog, int32_t *num_luts, int32_t *peak_live,
                     int32_t *num_gates) {
    return es_map_stats_k(prog, 0, num_luts, peak_live, num_gates, nullptr);
}

int32_t es_map_stats_k(const es_prog *prog, int32_t k, int32_t *num_luts, int32_t *peak_live,
                       int32_t *num_gates, int32_t *cof_pis) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    if (num_luts) *num_luts = (int32_t)net.luts.size();
    if (peak_live) *peak_live = net.peak_live;
    if (num_gates) *num_gates = net.num_gates;
    if (cof_pis)
        for (int i = 0; i < (int)net.cof_pis.size() && i < k; ++i) cof_pis[i] = net.cof_pis[i];
    return ES_OK;
}

int32_t es_map_pipes(const es_prog *prog, int32_t *lop3, int32_t *imad) {
    return es_map_pipes_k(prog, 0, lop3, imad);
}

int32_t es_map_pipes_k(const es_prog *prog, int32_t k, int32_t *lop3, int32_t *imad) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    const std::string body = emit_body_ptx(net, {"%o", "%c"}, "%lo", "%hi", "%one");
    int nl = 0, ni = 0;
    for (size_t p = 0; (p = body.find("lop3.b32 %esq", p)) != std::string::npos; ++p) ++nl;
    for (size_t p = 0; (p = body.find("mad.lo.s32 %esq", p)) != std::string::npos; ++p) ++ni;
    if (lop3) *lop3 = nl;
    if (imad) *imad = ni;
    return ES_OK;
}

int64_t es_emit_body_k(const es_prog *prog, int32_t k, int32_t spill_budget, int32_t block_threads,
                       int32_t *slots, char *buf, int64_t cap) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    const bool multi = net.outs.size() > 1 || !net.cof_pis.empty();
    std::string body = emit_body_ptx(net, multi ? std::vector<std::string>{"%o", "%c"} : std::vector<std::string>{"%o"},
                                     "%lo", "%hi", "%one");
    SpillStats ss;
    if (spill_budget > 0) body = spill_body(body, spill_budget, block_threads > 0 ? block_threads : 256, &ss);
    if (slots) *slots = ss.slots;
    const int64_t n = (int64_t)body.size() + 1;
    if (!buf) return n;
    if (cap < n) { set_error("buffer too small"); return ES_E_BAD_ARG; }
    memcpy(buf, body.c_str(), (size_t)n);
    return n;
}

int64_t es_sass_cubin(const es_prog *prog, int32_t k, int32_t block_threads, int32_t *stats, char *buf,
                      int64_t cap) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    std::vector<char> cubin;
    SassStats ss;
    std::string err;
    if (!sass_direct_cubin(net, block_threads, &cubin, &ss, &err)) { set_error(err); return ES_E_BAD_ARG; }
    if (stats) {
        stats[0] = ss.instrs;
        stats[1] = ss.lop3;
        stats[2] = ss.imad;
        stats[3] = ss.regs_peak;
        stats[4] = ss.cycles;
        stats[5] = ss.reg_lo;
        stats[6] = ss.reg_hi;
        stats[7] = ss.reg_o0;
        stats[8] = ss.reg_o1;
    }
    const int64_t n = (int64_t)cubin.size();
    if (!buf) return n;
    if (cap < n) { set_error("buffer too small"); return ES_E_BAD_ARG; }
    memcpy(buf, cubin.data(), (size_t)n);
    return n;
}

int64_t es_k4_cubin(const es_prog *progs, int32_t n, const int32_t *cof_k, int32_t variant, int32_t *stats,
                    char *buf, int64_t cap) {
    if (!progs || n <= 0 || variant < 0 || variant >= k4_variants() || n > k4_max_bodies(variant)) {
        set_error("bad argument");
        return ES_E_BAD_ARG;
    }
    std::vector<std::vector<uint64_t>> code(n);
    SassStats ss;
    for (int i = 0; i < n; ++i) {
        LutNet net;
        int rc = map_prog(&progs[i], &net, cof_k ? cof_k[i] : 0);
        if (rc != ES_OK) return rc;
        std::string err;
        int used = 0;
        if (!k4_body(net, variant, &code[i], &ss, &used, &err)) { set_error(err); return ES_E_BAD_ARG; }
        if (stats) stats[4 * i] = ss.instrs;
    }
    if (stats) {
        stats[4 * n] = ss.reg_lo;
        stats[4 * n + 1] = ss.reg_hi;
        stats[4 * n + 2] = ss.reg_o0;
        stats[4 * n + 3] = ss.reg_o1;
    }
    std::vector<const std::vector<uint64_t> *> bodies;
    for (auto &c : code) bodies.push_back(&c);
    std::vector<char> cubin;
    std::vector<uint32_t> entry;
    std::string err;
    if (!k4_module(bodies, variant, &cubin, &entry, &err)) { set_error(err); return ES_E_BAD_ARG; }
    const int64_t sz = (int64_t)cubin.size();
    if (!buf) return sz;
    if (cap < sz) { set_error("buffer too small"); return ES_E_BAD_ARG; }
    memcpy(buf, cubin.data(), (size_t)sz);
    return sz;
}

int32_t es_map_eval(const es_prog *prog, uint64_t w0, uint64_t nw, uint32_t *out_words) {
    return es_map_eval_k(prog, 0, w0, nw, out_words);
}

int32_t es_map_eval_k(const es_prog *prog, int32_t k, uint64_t w0, uint64_t nw, uint32_t *out_words) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    eval_lutnet(net, w0, nw, out_words);
    return ES_OK;
}

int32_t es_map_stats_kc(const es_prog *prog, int32_t k, int32_t copies, int32_t *num_luts,
                        int32_t *peak_live) {
    LutNet net;
    int rc = map_prog(prog, &net, k, copies);
    if (rc != ES_OK) return rc;
    if (num_luts) *num_luts = (int32_t)net.luts.size();
    if (peak_live) *peak_live = net.peak_live;
    return ES_OK;
}

int32_t es_map_eval_kc(const es_prog *prog, int32_t k, int32_t copies, uint64_t w0, uint64_t nw,
                       uint32_t *out_words) {
    LutNet net;
    int rc = map_prog(prog, &net, k, copies);
    if (rc != ES_OK) return rc;
    eval_lutnet(net, w0, nw, out_words);
    return ES_OK;
}

int32_t es_k2_stats(const es_prog *prog, int32_t *num_gates, int32_t *num_slots,
                    int32_t *stores, int32_t *acc_reads) {
    if (!prog || prog->num_instrs < 1) { set_error("empty program"); return ES_E_BAD_PROGRAM; }
    Dag dag;
    std::string err;
    int rc = build_dag(*prog, &dag, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    K2Prog kp;
    build_k2prog_auto(dag, &kp);
    int st = 0, acc = 0;
    for (const K2Gate &g : kp.gates) {
        st += (g.ctl & K2_STORE) != 0;
        acc += (g.ctl & K2_A_ACC) != 0;
    }
    if (num_gates) *num_gates = kp.n_gates;
    if (num_slots) *num_slots = kp.num_slots;
    if (stores) *stores = st;
    if (acc_reads) *acc_reads = acc;
    return ES_OK;
}

int32_t es_k2_eval(const es_prog *prog, uint64_t w0, uint64_t nw, uint32_t *out_words) {
    if (!prog || prog->num_instrs < 1) { set_error("empty program"); return ES_E_BAD_PROGRAM; }
    Dag dag;
    std::string err;
    int rc = build_dag(*prog, &dag, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    K2Prog kp;
    build_k2prog_auto(dag, &kp);
    eval_k2prog(kp, w0, nw, out_words);
    return ES_OK;
}

int32_t es_k2_eval_k(const es_prog *prog, int32_t k, uint64_t w0, uint64_t nw, uint32_t *out_words) {
    if (!prog || prog->num_instrs < 1) { set_error("empty program"); return ES_E_BAD_PROGRAM; }
    if (k < 0 || k > kK2MaxCofactorPis) { set_error("cofactor PIs must be 0..6"); return ES_E_BAD_ARG; }
    Dag dag;
    std::string err;
    int rc = build_dag(*prog, &dag, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    K2Prog kp;
    build_k2prog_k(dag, k, &kp);
    if ((int)kp.cof_pis.size() != k) { set_error("fewer word PIs than cofactor PIs"); return ES_E_BAD_ARG; }
    eval_k2prog(kp, w0, nw, out_words);
    return ES_OK;
}

int32_t es_k2_cofactor_pis(const es_prog *prog) {
    if (!prog || prog->num_instrs < 1) { set_error("empty program"); return ES_E_BAD_PROGRAM; }
    Dag dag;
    std::string err;
    int rc = build_dag(*prog, &dag, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    K2Prog kp;
    build_k2prog_auto(dag, &kp);
    return (int32_t)kp.cof_pis.size();
}

int64_t es_emit_ptx(const es_prog *prog, int32_t block_threads, char *buf, int64_t cap) {
    return es_emit_ptx_k(prog, 0, block_threads, buf, cap);
}

int64_t es_emit_ptx_k(const es_prog *prog, int32_t k, int32_t block_threads, char *buf, int64_t cap) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    std::string ptx, err;
    if (!splice_body(net, block_threads != 0 ? block_threads : 256, &ptx, &err)) {
        set_error(err);
        return ES_E_BAD_ARG;
    }
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, (int64_t)ptx.size());
        std::memcpy(buf, ptx.data(), (size_t)n);
        buf[n] = '\0';
    }
    return (int64_t)ptx.size() + 1;
}

int64_t es_jit_check(const es_prog *prog, int32_t block_threads, int32_t *regs_per_thread,
                     int32_t *spill_bytes, char *log, int64_t log_cap) {
    return es_jit_check_k(prog, 0, block_threads, regs_per_thread, spill_bytes, log, log_cap);
}

int64_t es_jit_check_k(const es_prog *prog, int32_t k, int32_t block_threads, int32_t *regs_per_thread,
                       int32_t *spill_bytes, char *log, int64_t log_cap) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    std::string ptx, err, info;
    if (!splice_body(net, block_threads != 0 ? block_threads : 256, &ptx, &err)) {
        set_error(err);
        return ES_E_BAD_ARG;
    }
    std::vector<char> cubin;
    rc = ptx_to_cubin(ptx, &cubin, &info, &err);
    if (rc != ES_OK) { set_error(err); return rc; }
    if (const char *dump = getenv("ES_DUMP_CUBIN")) {  // for cuobjdump -sass
        if (FILE *f = fopen(dump, "wb")) { fwrite(cubin.data(), 1, cubin.size(), f); fclose(f); }
    }
    int regs = -1, spill = 0;
    parse_ptxas_info(info, &regs, &spill);
    if (regs_per_thread) *regs_per_thread = regs;
    if (spill_bytes) *spill_bytes = spill;
    if (log && log_cap > 0) {
        const int64_t n = std::min<int64_t>(log_cap - 1, (int64_t)info.size());
        std::memcpy(log, info.data(), (size_t)n);
        log[n] = '\0';
    }
    return (int64_t)cubin.size();
}

int64_t es_jit_check_split(const es_prog *prog, int32_t k, int32_t parts, int32_t block_threads,
                           int32_t *regs_per_thread, int32_t *smem_bytes, int32_t *slots, int32_t *loads,
                           double *ms) {
    LutNet net;
    int rc = map_prog(prog, &net, k);
    if (rc != ES_OK) return rc;
    const int threads = block_threads != 0 ? block_threads : 128;
    const double t0 = now_ms();
    std::string skel, err, info;
    std::vector<std::string> phases;
    int smem = 0;
    if (!splice_split(net, threads, parts, &skel, &phases, &err, &smem)) {
        set_error(err);
        return ES_E_BAD_ARG;
    }
    if (const char *dir = getenv("ES_DUMP_SPLIT")) {  // the modules, for ptxas / cuobjdump by hand
        for (size_t m = 0; m <= phases.size(); ++m) {
            const std::string path = std::string(dir) + "/mod" + std::to_string(m) + ".ptx";
            if (FILE *f = fopen(path.c_str(), "w")) {
                const std::string &txt = m == 0 ? skel : phases[m - 1];
                fwrite(txt.data(), 1, txt.size(), f);
                fclose(f);
            }
        }
    }
    std::vector<char> cubin;
    rc = split_to_cubin(skel, phases, &cubin, &info, &err, 1);
    if (rc != ES_OK) { set_error(err); return rc; }
    if (ms) *ms = now_ms() - t0;
    if (const char *dump = getenv("ES_DUMP_CUBIN")) {
        if (FILE *f = fopen(dump, "wb")) { fwrite(cubin.data(), 1, cubin.size(), f); fclose(f); }
    }
    int regs = -1, spill = 0;
    parse_ptxas_info(info, &regs, &spill);
    if (regs_per_thread) *regs_per_thread = regs;
    if (smem_bytes) *smem_bytes = smem;
    if (slots) *slots = smem / (threads * 4);
    if (loads) {  // slot loads per iteration: count them in the phase text
        int nl = 0;
        for (const std::string &ph : phases)
            for (size_t p = ph.find("ld.shared.b32"); p != std::string::npos; p = ph.find("ld.shared.b32", p + 1)) ++nl;
        *loads = nl;
    }
    return (int64_t)cubin.size();
}

int32_t es_sim(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
               const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
               uint64_t *node_words, double *device_ms) {
    if ((num_gates > 0 && (!kind || !in0 || !in1)) || (num_pis > 0 && !pi_words) || !node_words) {
        set_error("null argument");
        return ES_E_BAD_ARG;
    }
    return sim_run(num_pis, num_gates, kind, in0, in1, pi_words, words, device, node_words, device_ms);
}

int32_t es_sim_ones(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
                    int64_t *ones, double *device_ms) {
    if ((num_gates > 0 && (!kind || !in0 || !in1)) || (num_pis > 0 && !pi_words) || !ones) {
        set_error("null argument");
        return ES_E_BAD_ARG;
    }
    return sim_ones(num_pis, num_gates, kind, in0, in1, pi_words, words, device, ones, device_ms);
}

int32_t es_sim_device(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                      const uint32_t *in1, const uint64_t *d_pi_words, int64_t words, void *stream,
                      uint64_t *d_node_words, void **prog_cache) {
    if ((num_gates > 0 && (!kind || !in0 || !in1)) || !d_node_words) { set_error("null argument"); return ES_E_BAD_ARG; }
    return sim_run_device(num_pis, num_gates, kind, in0, in1, d_pi_words, words, stream, d_node_words,
                          prog_cache);
}

void es_sim_prog_free(void *prog_cache) { sim_prog_free(prog_cache); }

int32_t es_sim_levels(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                     const uint32_t *in1) {
    if (num_gates > 0 && (!kind || !in0 || !in1)) { set_error("null argument"); return ES_E_BAD_ARG; }
    return sim_levels(num_pis, num_gates, kind, in0, in1);
}

int32_t es_sim_classes(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                       const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
                       int32_t *class_id, uint8_t *polarity, int32_t *n_classes, double *device_ms) {
    if ((num_gates > 0 && (!kind || !in0 || !in1)) || (num_pis > 0 && !pi_words)) {
        set_error("null argument");
        return ES_E_BAD_ARG;
    }
    return sim_classes(num_pis, num_gates, kind, in0, in1, pi_words, words, device, class_id, polarity,
                       n_classes, device_ms);
}

int32_t es_aiger_parse(const uint8_t *data, int64_t len, int32_t detect_xors, es_xag **out) {
    if ((!data && len > 0) || len < 0 || !out) { set_error("bad argument"); return ES_E_BAD_ARG; }
    XagC *x = nullptr;
    static const uint8_t kEmpty = 0;
    const int rc = aiger_parse(data ? data : &kEmpty, len, detect_xors, &x);
    *out = (es_xag *)x;
    return rc;
}

int32_t es_detect_xors(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                       const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits,
                       es_xag **out) {
    if (!out || num_pis < 0 || num_gates < 0 || num_outputs < 0 ||
        (num_gates > 0 && (!kind || !in0 || !in1)) || (num_outputs > 0 && !out_lits)) {
        set_error("bad argument");
        return ES_E_BAD_ARG;
    }
    XagC *x = nullptr;
    const int rc = xag_detect_xors(num_pis, num_gates, kind, in0, in1, num_outputs, out_lits, &x);
    *out = (es_xag *)x;
    return rc;
}

int32_t es_xag_size(const es_xag *xp, int32_t *num_pis, int32_t *num_gates, int32_t *num_outputs) {
    const XagC *x = (const XagC *)xp;
    if (!x) { set_error("null xag"); return ES_E_BAD_ARG; }
    if (num_pis) *num_pis = x->num_pis;
    if (num_gates) *num_gates = (int32_t)x->kind.size();
    if (num_outputs) *num_outputs = (int32_t)x->outs.size();
    return ES_OK;
}

int32_t es_xag_read(const es_xag *xp, uint8_t *kind, uint32_t *in0, uint32_t *in1, uint32_t *out_lits) {
    const XagC *x = (const XagC *)xp;
    if (!x) { set_error("null xag"); return ES_E_BAD_ARG; }
    if (kind) std::memcpy(kind, x->kind.data(), x->kind.size());
    if (in0) std::memcpy(in0, x->in0.data(), 4 * x->in0.size());
    if (in1) std::memcpy(in1, x->in1.data(), 4 * x->in1.size());
    if (out_lits) std::memcpy(out_lits, x->outs.data(), 4 * x->outs.size());
    return ES_OK;
}

void es_xag_free(es_xag *xp) { delete (XagC *)xp; }

int64_t es_aiger_write(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                       const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits, char *buf,
                       int64_t cap) {
    if (num_pis < 0 || num_gates < 0 || num_outputs < 0 || (num_gates > 0 && (!kind || !in0 || !in1)) ||
        (num_outputs > 0 && !out_lits)) {
        set_error("bad argument");
        return ES_E_BAD_ARG;
    }
    return aiger_write(num_pis, num_gates, kind, in0, in1, num_outputs, out_lits, buf, cap);
}

int32_t es_alu_peak(int32_t device, double *lane_ops_per_s, double *ms) {
    if (!lane_ops_per_s) return ES_E_BAD_ARG;
    return alu_peak(device, lane_ops_per_s, ms);
}

int32_t es_fma_peak(int32_t device, double *lane_ops_per_s, double *ms) {
    if (!lane_ops_per_s) return ES_E_BAD_ARG;
    return fma_peak(device, lane_ops_per_s, ms);
}

int32_t es_smem_peak(int32_t device, double *bytes_per_s, double *ms) {
    if (!bytes_per_s) return ES_E_BAD_ARG;
    return smem_peak(device, bytes_per_s, ms);
}

int32_t es_batch_extract(int32_t num_pis, int32_t num_gates, const uint8_t *kind,
                         const uint32_t *in0, const uint32_t *in1, int32_t n_merges,
                         const int32_t *merge_node, const uint32_t *merge_lit, int32_t n_pairs,
                         const int32_t *a, const int32_t *b, const uint8_t *polarity,
                         int32_t n_threads, es_batch **out) {
    if (!out || n_pairs < 0 || num_pis < 0 || num_gates < 0) { set_error("bad argument"); return ES_E_BAD_ARG; }
    Batch *bt = new Batch();
    std::string err;
    int rc = extract_compile(num_pis, num_gates, kind, in0, in1, n_merges, merge_node, merge_lit,
                             n_pairs, a, b, polarity, n_threads, &bt->subs, &err);
    if (rc != ES_OK) { set_error(err); delete bt; return rc; }
    *out = (es_batch *)bt;
    return ES_OK;
}

int32_t es_batch_prepare(es_batch *bp, int32_t n_threads) {
    Batch *bt = (Batch *)bp;
    if (!bt) { set_error("bad argument"); return ES_E_BAD_ARG; }
    const int rc = prepare_k2(bt->subs, n_threads);
    if (rc != ES_OK) { set_error("malformed sub-miter program"); return rc; }
    // and the K4 straight-line bodies of the jobs with enough words
    std::vector<es_prog> progs(bt->subs.size());
    std::vector<const K2Prog *> kps(bt->subs.size(), nullptr);
    for (size_t i = 0; i < bt->subs.size(); ++i) {
        if (bt->subs[i].too_many_inputs) continue;
        progs[i] = bt->subs[i].view();
        kps[i] = &bt->subs[i].k2;
    }
    k4_prebuild((int)progs.size(), progs.data(), kps.data());
    return ES_OK;
}

int32_t es_xag_eval(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, uint32_t out_lit, uint64_t pattern) {
    if (num_pis < 0 || num_pis > 64 || num_gates < 0 || (num_gates > 0 && (!kind || !in0 || !in1))) {
        set_error("bad argument");
        return ES_E_BAD_ARG;
    }
    const uint32_t nn = 1u + (uint32_t)num_pis + (uint32_t)num_gates;
    std::vector<uint8_t> v(nn, 0);
    for (int i = 0; i < num_pis; ++i) v[1 + i] = (pattern >> i) & 1;
    for (int g = 0; g < num_gates; ++g) {
        const uint32_t a = in0[g] >> 1, b = in1[g] >> 1;
        if (a >= 1u + num_pis + g || b >= 1u + num_pis + g) { set_error("XAG not topological"); return ES_E_BAD_PROGRAM; }
        const uint8_t x = v[a] ^ (in0[g] & 1), y = v[b] ^ (in1[g] & 1);
        v[1 + num_pis + g] = kind[g] ? (x ^ y) : (x & y);
    }
    if ((out_lit >> 1) >= nn) { set_error("output literal out of range"); return ES_E_BAD_ARG; }
    return v[out_lit >> 1] ^ (out_lit & 1);
}

int32_t es_batch_k2_stats(const es_batch *bp, int32_t *num_slots, int32_t *num_records,
                          int32_t *cofactor_pis) {
    const Batch *bt = (const Batch *)bp;
    if (!bt) { set_error("bad argument"); return ES_E_BAD_ARG; }
    for (size_t i = 0; i < bt->subs.size(); ++i) {
        const SubMiterC &s = bt->subs[i];
        const bool ok = s.k2_ready;
        if (num_slots) num_slots[i] = ok ? s.k2.num_slots : -1;
        if (num_records) num_records[i] = ok ? (int32_t)s.k2.gates.size() : -1;
        if (cofactor_pis) cofactor_pis[i] = ok ? (int32_t)s.k2.cof_pis.size() : -1;
    }
    return ES_OK;
}

int32_t es_batch_k2_traffic(const es_batch *bp, int32_t *loads, int32_t *stores) {
    const Batch *bt = (const Batch *)bp;
    if (!bt) { set_error("bad argument"); return ES_E_BAD_ARG; }
    for (size_t i = 0; i < bt->subs.size(); ++i) {
        const SubMiterC &s = bt->subs[i];
        const bool ok = s.k2_ready;
        // per pass over the records: operand loads, result stores, and the
        // PI words stored into their slots at the start of every pass
        if (loads) loads[i] = ok ? s.k2.loads : -1;
        if (stores) stores[i] = ok ? s.k2.stores + s.num_pis - (int32_t)s.k2.cof_pis.size() : -1;
    }
    return ES_OK;
}

int32_t es_batch_size(const es_batch *bp) { return bp ? (int32_t)((const Batch *)bp)->subs.size() : ES_E_BAD_ARG; }

int32_t es_batch_info(const es_batch *bp, int32_t i, int32_t *num_pis, int32_t *num_gates,
                      uint64_t *hash, int32_t *num_instrs, int32_t *num_registers, int32_t *G) {
    const Batch *bt = (const Batch *)bp;
    if (!bt || i < 0 || i >= (int32_t)bt->subs.size()) { set_error("index out of range"); return ES_E_BAD_ARG; }
    const SubMiterC &s = bt->subs[i];
    if (num_pis) *num_pis = s.num_pis;
    if (num_gates) *num_gates = (int32_t)s.kind.size();
    if (hash) *hash = s.hash;
    if (num_instrs) *num_instrs = s.too_many_inputs ? 0 : (int32_t)s.op.size();
    if (num_registers) *num_registers = s.num_registers;
    if (G) *G = s.G;
    return s.too_many_inputs ? ES_E_TOO_MANY_INPUTS : ES_OK;
}

int32_t es_batch_table(const es_batch *bp, int32_t *num_pis, int32_t *num_gates, int32_t *G,
                       uint64_t *hash) {
    const Batch *bt = (const Batch *)bp;
    if (!bt) { set_error("bad argument"); return ES_E_BAD_ARG; }
    for (size_t i = 0; i < bt->subs.size(); ++i) {
        const SubMiterC &s = bt->subs[i];
        if (num_pis) num_pis[i] = s.num_pis;
        if (num_gates) num_gates[i] = (int32_t)s.kind.size();
        if (G) G[i] = s.G;
        if (hash) hash[i] = s.hash;
    }
    return ES_OK;
}

int32_t es_batch_xag(const es_batch *bp, int32_t i, uint8_t *kind, uint32_t *in0, uint32_t *in1,
                     uint32_t *out_lit, int32_t *pi_map) {
    const Batch *bt = (const Batch *)bp;
    if (!bt || i < 0 || i >= (int32_t)bt->subs.size()) { set_error("index out of range"); return ES_E_BAD_ARG; }
    const SubMiterC &s = bt->subs[i];
    if (kind) std::memcpy(kind, s.kind.data(), s.kind.size());
    if (in0) std::memcpy(in0, s.in0.data(), 4 * s.in0.size());
    if (in1) std::memcpy(in1, s.in1.data(), 4 * s.in1.size());
    if (out_lit) *out_lit = s.out_lit;
    if (pi_map) std::memcpy(pi_map, s.pi_map.data(), 4 * s.pi_map.size());
    return ES_OK;
}

int32_t es_batch_select(es_batch *bp, int32_t n, const int32_t *idx) {
    Batch *bt = (Batch *)bp;
    if (!bt || n < 0) { set_error("bad argument"); return ES_E_BAD_ARG; }
    std::vector<SubMiterC> keep;
    keep.reserve(n);
    for (int k = 0; k < n; ++k) {
        if (idx[k] < 0 || idx[k] >= (int32_t)bt->subs.size()) { set_error("index out of range"); return ES_E_BAD_ARG; }
        keep.push_back(bt->subs[idx[k]]);
    }
    bt->subs.swap(keep);
    return ES_OK;
}

int32_t es_batch_run(es_batch *bp, const es_run_opts *opts, es_result *outs) {
    Batch *bt = (Batch *)bp;
    if (!bt || !outs) { set_error("bad argument"); return ES_E_BAD_ARG; }
    const int n = (int)bt->subs.size();
    const double t_in = now_ms();
    // jobs worth a JIT kernel of their own (>= kBatchJitWork gate-patterns,
    // ~20 ms and up in the interpreter) run through K1, the rest through one
    // batched K2 launch
    constexpr double kBatchJitWork = 2e12;
    std::vector<es_prog> progs, big_progs;
    std::vector<const K2Prog *> kps;
    std::vector<int> where, big_where;
    bool force_interp = opts && opts->engine == ES_ENGINE_INTERP;
    for (int i = 0; i < n; ++i) {
        std::memset(&outs[i], 0, sizeof(es_result));
        if (bt->subs[i].too_many_inputs) { outs[i].verdict = ES_BUDGET_EXCEEDED; outs[i].reason = -1; continue; }
        const es_prog v = bt->subs[i].view();
        if (!force_interp && (double)bt->subs[i].G * std::ldexp(1.0, v.num_pis) >= kBatchJitWork) {
            big_progs.push_back(v);
            big_where.push_back(i);
            continue;
        }
        progs.push_back(v);
        where.push_back(i);
    }
    const double t0 = now_ms();
    // no-op once es_batch_prepare ran; cofactor_pis NONE skips the depth search
    const bool search = !(opts && opts->cofactor_pis == ES_COFACTOR_NONE);
    int prc = prepare_k2(bt->subs, 0, &where, search);
    if (prc != ES_OK) { set_error("malformed sub-miter program"); return prc; }
    kps.reserve(where.size());
    for (int i : where) kps.push_back(&bt->subs[i].k2);
    std::vector<es_result> rs(progs.size()), big_rs(big_progs.size());
    const double t1 = now_ms();
    int rc = progs.empty() ? ES_OK : run_batch((int)progs.size(), progs.data(), opts, rs.data(), kps.data());
    if (rc != ES_OK) return rc;
    const double t2 = now_ms();
    if (!big_progs.empty()) {
        es_run_opts ob{};
        if (opts) ob = *opts;
        if (ob.budget_s >= 0 && opts) ob.budget_s = std::max(0.0, ob.budget_s - 1e-3 * (t2 - t0));
        rc = run_batch_jit((int)big_progs.size(), big_progs.data(), &ob, big_rs.data());
        if (rc != ES_OK) return rc;
    }
    if (getenv("ES_VERBOSE"))
        fprintf(stderr, "[es batch] jobs=%d (K1 %zu) split=%.2fms prep=%.2fms K2=%.2fms K1=%.2fms\n", n,
                big_progs.size(), t0 - t_in, t1 - t0, t2 - t1, now_ms() - t2);
    for (size_t k = 0; k < big_where.size(); ++k) {
        where.push_back(big_where[k]);
        rs.push_back(big_rs[k]);
    }
    // re-check every witness on its sub-miter (es.py:360), on all host cores
    std::atomic<int> bad_job{-1};
    parallel_for((int)where.size(), [&](int k) {
        outs[where[k]] = rs[k];
        if (rs[k].verdict == ES_COUNTEREXAMPLE && evaluate_sub(bt->subs[where[k]], rs[k].witness_index) != 1) {
            int none = -1;
            bad_job.compare_exchange_strong(none, where[k]);
        }
    });
    if (bad_job.load() >= 0) {
        set_error("exhaustive-simulation witness failed re-check (job " + std::to_string(bad_job.load()) + ")");
        return ES_E_WITNESS;
    }
    if (getenv("ES_VERBOSE")) fprintf(stderr, "[es batch] total %.2fms\n", now_ms() - t_in);
    return ES_OK;
}

int32_t es_batch_merge(es_batch *dst, es_batch *src) {
    Batch *d = (Batch *)dst, *s = (Batch *)src;
    if (!d || !s || d == s) { set_error("bad argument"); return ES_E_BAD_ARG; }
    for (auto &x : s->subs) d->subs.push_back(std::move(x));
    s->subs.clear();
    return ES_OK;
}

void es_batch_free(es_batch *bp) { delete (Batch *)bp; }

int32_t es_ipc_alloc(int32_t device, void **dev_ptr, uint8_t *handle64) {
    if (!dev_ptr || !handle64) return ES_E_BAD_ARG;
    return ipc_alloc(device, dev_ptr, handle64);
}

int32_t es_ipc_open(int32_t device, const uint8_t *handle64, void **dev_ptr) {
    if (!dev_ptr || !handle64) return ES_E_BAD_ARG;
    return ipc_open(device, handle64, dev_ptr);
}

int32_t es_ipc_close(int32_t device, void *dev_ptr, int32_t owner) {
    return ipc_close(device, dev_ptr, owner);
}

int32_t es_word_write(int32_t device, void *dev_ptr, uint64_t value) {
    return word_io(device, dev_ptr, &value, 1);
}

int32_t es_peer_arm(void *stream, void *word_dev) {
    if (!word_dev) { set_error("null word"); return ES_E_BAD_ARG; }
    return peer_arm(stream, word_dev);
}

int32_t es_peer_arrive_wait(void *stream, void *word_dev, int32_t world, void *out_dev) {
    if (!word_dev || !out_dev) { set_error("null argument"); return ES_E_BAD_ARG; }
    return peer_arrive_wait(stream, word_dev, world, out_dev);
}

int32_t es_word_read(int32_t device, void *dev_ptr, uint64_t *value) {
    if (!value) return ES_E_BAD_ARG;
    return word_io(device, dev_ptr, value, 0);
}

const char *es_last_error(void) { return t_err.c_str(); }

const char *es_version(void) { return "es_b200 0.1 (sm_100a)"; }

void es_shutdown(void) { runtime_shutdown(); }

}  // extern "C"
