// es_jit.cpp -- per-program JIT of K1: splice the generated LOP3 body into the
// hand-written skeleton PTX (k1_skeleton.cu), compile it to sm_100a SASS with
// the in-process PTX compiler (libnvptxcompiler_static, no driver JIT, no
// GPU needed), load it with cudaLibraryLoadData.  Modules are cached by a
// hash of the final PTX, so a program is compiled once per process.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <sys/stat.h>
#include <unistd.h>
#include <atomic>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>
#include <nvJitLink.h>
#include <nvPTXCompiler.h>
#include <thread>

#include "es_jit.h"
#include "es_nvtx.h"

namespace es {

#include "k1_skeleton_ptx.inc"  // kK1Ptx<threads>_<copies>

static const char *skeleton_for(int threads, int copies) {
    const bool multi = copies > 1;
    switch (threads) {
        case 128: return multi ? kK1Ptx128_1 : kK1Ptx128_0;
        case 256: return multi ? kK1Ptx256_1 : kK1Ptx256_0;
        case 512: return multi ? nullptr : kK1Ptx512_0;
        default: return nullptr;
    }
}

bool splice_body(const LutNet &net, int threads, std::string *ptx, std::string *err,
                 int *region_bytes) {
    if (region_bytes) *region_bytes = 0;
    // the multi-copy skeleton whenever there are cofactor PIs (it inserts
    // their bits into pattern indices), even for a one-copy restricted variant
    const int copies = net.cof_pis.empty() ? (int)net.outs.size() : std::max(2, (int)net.outs.size());
    const char *sk = skeleton_for(threads, copies);
    if (!sk) {
        *err = "unsupported K1 variant: " + std::to_string(threads) + " threads x " +
               std::to_string(copies) + " copies";
        return false;
    }
    std::string s(sk);
    const std::string marker = "// ES_BODY ";
    size_t at = s.find(marker);
    if (at == std::string::npos || s.find(marker, at + 1) != std::string::npos) {
        *err = "K1 skeleton must contain exactly one ES_BODY marker";
        return false;
    }
    size_t eol = s.find('\n', at);
    std::istringstream in(s.substr(at + marker.size(), eol - at - marker.size()));
    std::vector<std::string> a;
    for (std::string t; in >> t;) a.push_back(t);
    const int nout = copies > 1 ? 2 : 1;  // (first failing word, its copy) or the output word
    if ((int)a.size() != nout + 3) {
        *err = "cannot parse ES_BODY operands (" + std::to_string(a.size()) + ")";
        return false;
    }
    const std::vector<std::string> outs(a.begin(), a.begin() + nout);
    std::string body = emit_body_ptx(net, outs, a[nout], a[nout + 1], a[nout + 2]);
    if (const char *e = getenv("ES_K1_SPILL_R")) {  // shared-memory overflow slots (es_spill.cpp)
        SpillStats ss;
        body = spill_body(body, atoi(e), threads, &ss);
        if (ss.slots > 0) {
            const size_t hdr = s.find('\n', s.find(".address_size 64")) + 1;
            s.insert(hdr, ".extern .shared .align 16 .b8 es_slots[];\n");
            at = s.find(marker);
            eol = s.find('\n', at);
            if (region_bytes) *region_bytes = ss.slots * threads * 4;
        }
        if (getenv("ES_VERBOSE"))
            fprintf(stderr, "[es] K1 spill budget %s: %d slots, %d loads, %d stores per iteration\n", e, ss.slots,
                    ss.loads, ss.stores);
    }
    s.replace(at, eol - at, body);
    if (const char *m = getenv("ES_MAXNREG")) {  // experiment: register cap for occupancy
        const size_t mt = s.find(".maxntid");
        if (mt != std::string::npos) s.insert(s.find('\n', mt) + 1, std::string(".maxnreg ") + m + "\n");
    }
    *ptx = std::move(s);
    return true;
}

// Split build (es_split.cpp): the skeleton with its body replaced by calls
// to `parts` phase functions, and the phase modules.  smem_bytes: the
// dynamic shared memory of the slot file.
bool splice_split(const LutNet &net, int threads, int parts, std::string *skel,
                  std::vector<std::string> *phases, std::string *err, int *smem_bytes) {
    const int copies = net.cof_pis.empty() ? (int)net.outs.size() : std::max(2, (int)net.outs.size());
    const char *sk = skeleton_for(threads, copies);
    if (!sk) { *err = "unsupported K1 variant"; return false; }
    std::string s(sk);
    const std::string marker = "// ES_BODY ";
    const size_t at = s.find(marker);
    const size_t hdr_end = s.find(".address_size 64");
    if (at == std::string::npos || hdr_end == std::string::npos) { *err = "bad K1 skeleton"; return false; }
    const size_t hdr_eol = s.find('\n', hdr_end);
    size_t eol = s.find('\n', at);
    std::istringstream in(s.substr(at + marker.size(), eol - at - marker.size()));
    std::vector<std::string> a;
    for (std::string t; in >> t;) a.push_back(t);
    const int nout = copies > 1 ? 2 : 1;
    if ((int)a.size() != nout + 3) { *err = "cannot parse ES_BODY operands"; return false; }
    SplitPtx sp;
    const std::string header = s.substr(0, hdr_eol + 1);
    if (!emit_split_ptx(net, threads, parts, header, std::vector<std::string>(a.begin(), a.begin() + nout),
                        a[nout], a[nout + 1], a[nout + 2], &sp)) {
        *err = "program too small to split into " + std::to_string(parts) + " phases";
        return false;
    }
    s.replace(at, eol - at, sp.call_body);
    s.insert(hdr_eol + 1, sp.decls);
    *skel = std::move(s);
    *phases = std::move(sp.phases);
    *smem_bytes = sp.slots * threads * 4;
    return true;
}

static uint64_t fnv1a(const std::string &s) {
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) { h ^= c; h *= 1099511628211ull; }
    return h;
}

static int effective_opt(int opt) {
    const char *e = getenv("ES_PTXAS_O");
    return e ? atoi(e) : opt;
}

int ptx_to_cubin(const std::string &ptx, std::vector<char> *cubin, std::string *info,
                 std::string *err, int opt, bool relocatable) {
    nvPTXCompilerHandle h = nullptr;
    if (nvPTXCompilerCreate(&h, ptx.size(), ptx.c_str()) != NVPTXCOMPILE_SUCCESS) {
        *err = "nvPTXCompilerCreate failed";
        return ES_E_CUDA;
    }
    std::vector<const char *> opts = {"--gpu-name=sm_100a", "--verbose"};
    std::string olev = "-O" + std::to_string(effective_opt(opt));
    opts.push_back(olev.c_str());
    if (relocatable) opts.push_back("-c");
    // experiments: extra ptxas options, space-separated (use with ES_JIT_CACHE=0)
    std::vector<std::string> extra;
    if (const char *e = getenv("ES_PTXAS_EXTRA")) {
        std::string cur;
        for (const char *c = e;; ++c) {
            if (*c == ' ' || *c == 0) { if (!cur.empty()) extra.push_back(cur); cur.clear(); if (!*c) break; }
            else cur += *c;
        }
    }
    for (const std::string &x : extra) opts.push_back(x.c_str());
    nvPTXCompileResult r = nvPTXCompilerCompile(h, (int)opts.size(), opts.data());
    size_t n = 0;
    if (r != NVPTXCOMPILE_SUCCESS) {
        nvPTXCompilerGetErrorLogSize(h, &n);
        std::string log(n, '\0');
        if (n) nvPTXCompilerGetErrorLog(h, &log[0]);
        *err = "PTX compile failed (" + std::to_string((int)r) + "): " + log;
        nvPTXCompilerDestroy(&h);
        return ES_E_CUDA;
    }
    nvPTXCompilerGetCompiledProgramSize(h, &n);
    cubin->resize(n);
    nvPTXCompilerGetCompiledProgram(h, cubin->data());
    size_t m = 0;
    nvPTXCompilerGetInfoLogSize(h, &m);
    info->assign(m, '\0');
    if (m) nvPTXCompilerGetInfoLog(h, &(*info)[0]);
    nvPTXCompilerDestroy(&h);
    return ES_OK;
}

void parse_ptxas_info(const std::string &info, int *regs, int *spill_bytes) {
    // "... Used 118 registers, ..." and "... N bytes spill stores, M bytes spill loads"
    *regs = -1;
    *spill_bytes = 0;
    size_t p = info.find("Used ");
    if (p != std::string::npos) *regs = atoi(info.c_str() + p + 5);
    p = info.find("bytes spill stores");
    if (p != std::string::npos) {
        size_t q = info.rfind(',', p);
        size_t start = q == std::string::npos ? 0 : q + 1;
        int st = atoi(info.c_str() + start);
        size_t r = info.find("bytes spill loads", p);
        int ld = 0;
        if (r != std::string::npos) {
            size_t q2 = info.rfind(',', r);
            ld = atoi(info.c_str() + (q2 == std::string::npos ? 0 : q2 + 1));
        }
        *spill_bytes = st + ld;
    }
}

namespace {
std::mutex g_jit_mu;
std::unordered_map<uint64_t, JitKernel *> g_cache;
std::vector<JitKernel *> g_uncached;  // kernels whose key collided with a resident entry

// On-disk cubin cache (the analogue of the reference's numba cache=True,
// es.py:175): a program compiled by one process is loaded by the next
// without running ptxas.  ES_JIT_CACHE=0 disables it; ES_JIT_CACHE_DIR
// overrides the directory (default $HOME/.cache/es_b200).  Entries are keyed
// by a hash of the final PTX and the PTX compiler version, and verified by a
// second hash and the PTX length on load.
std::string disk_cache_dir() {
    const char *off = getenv("ES_JIT_CACHE");
    if (off && std::string(off) == "0") return "";
    if (const char *d = getenv("ES_JIT_CACHE_DIR")) return d;
    const char *home = getenv("HOME");
    return home ? std::string(home) + "/.cache/es_b200" : "";
}

uint64_t second_hash(const std::string &s) {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ull + (h >> 27);
    return h;
}

std::string ptxc_version() {
    unsigned major = 0, minor = 0;
    nvPTXCompilerGetVersion(&major, &minor);
    return std::to_string(major) + "." + std::to_string(minor);
}

std::string entry_path(const std::string &dir, uint64_t key) {
    char name[64];
    snprintf(name, sizeof name, "/%016llx.esbin", (unsigned long long)key);
    return dir + name;
}

struct DiskHeader {
    char magic[8];
    uint64_t h2;
    uint64_t ptx_len;
    uint32_t info_len;
    uint32_t cubin_len;
};

bool disk_load(const std::string &dir, uint64_t key, const std::string &ptx, std::vector<char> *cubin,
               std::string *info) {
    if (dir.empty()) return false;
    FILE *f = fopen(entry_path(dir, key).c_str(), "rb");
    if (!f) return false;
    DiskHeader h{};
    bool ok = fread(&h, sizeof h, 1, f) == 1 && memcmp(h.magic, "ESBIN01", 8) == 0 &&
              h.h2 == second_hash(ptx) && h.ptx_len == ptx.size() && h.cubin_len > 0 &&
              h.cubin_len < (1u << 30) && h.info_len < (1u << 20);
    if (ok) {
        info->resize(h.info_len);
        cubin->resize(h.cubin_len);
        ok = (h.info_len == 0 || fread(&(*info)[0], 1, h.info_len, f) == h.info_len) &&
             fread(cubin->data(), 1, h.cubin_len, f) == h.cubin_len;
    }
    fclose(f);
    return ok;
}

void disk_store(const std::string &dir, uint64_t key, const std::string &ptx, const std::vector<char> &cubin,
                const std::string &info) {
    if (dir.empty()) return;
    std::string cmd = dir;  // mkdir -p
    for (size_t i = 1; i <= cmd.size(); ++i)
        if (i == cmd.size() || cmd[i] == '/') mkdir(cmd.substr(0, i).c_str(), 0755);
    const std::string path = entry_path(dir, key);
    const std::string tmp = path + ".tmp" + std::to_string((unsigned long long)getpid());
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) return;
    DiskHeader h{};
    memcpy(h.magic, "ESBIN01", 8);
    h.h2 = second_hash(ptx);
    h.ptx_len = ptx.size();
    h.info_len = (uint32_t)info.size();
    h.cubin_len = (uint32_t)cubin.size();
    const bool ok = fwrite(&h, sizeof h, 1, f) == 1 && fwrite(info.data(), 1, info.size(), f) == info.size() &&
                    fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
    fclose(f);
    if (ok) rename(tmp.c_str(), path.c_str());  // atomic publish
    else remove(tmp.c_str());
}
}  // namespace

// Split build: the skeleton and the phase modules compiled relocatable on
// parallel host threads (largest first), then linked by nvJitLink.  `info`
// gets a ptxas-style line with the largest register count and the summed
// spill bytes of the modules.
int split_to_cubin(const std::string &skel, const std::vector<std::string> &phases, std::vector<char> *cubin,
                   std::string *info, std::string *err, int opt) {
    const int M = 1 + (int)phases.size();
    std::vector<std::vector<char>> objs(M);
    std::vector<std::string> infos(M), errs(M);
    std::vector<int> rcs(M, ES_OK);
    std::atomic<int> next{0};
    auto work = [&]() {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= M) return;
            const int m = (i + 1) % M;  // phases first, the small skeleton last
            const double t0 = now_ms();
            rcs[m] = ptx_to_cubin(m == 0 ? skel : phases[m - 1], &objs[m], &infos[m], &errs[m], opt, true);
            if (getenv("ES_VERBOSE"))
                fprintf(stderr, "[es] split module %d: %.1f ms (%.1f .. %.1f)\n", m, now_ms() - t0, t0, now_ms());
        }
    };
    const int nt = std::min<int>(M, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int q = 1; q < nt; ++q) th.emplace_back(work);
    work();
    for (auto &x : th) x.join();
    int regs = 0, spill = 0;
    for (int m = 0; m < M; ++m) {
        if (rcs[m] != ES_OK) { *err = "split module " + std::to_string(m) + ": " + errs[m]; return rcs[m]; }
        int r = 0, sb = 0;
        parse_ptxas_info(infos[m], &r, &sb);
        regs = std::max(regs, r);
        spill += sb;
    }
    const double tl = now_ms();
    nvJitLinkHandle h = nullptr;
    const char *lopts[] = {"-arch=sm_100a"};
    if (nvJitLinkCreate(&h, 1, lopts) != NVJITLINK_SUCCESS) { *err = "nvJitLinkCreate failed"; return ES_E_CUDA; }
    nvJitLinkResult lr = NVJITLINK_SUCCESS;
    for (int m = 0; m < M && lr == NVJITLINK_SUCCESS; ++m) {
        const std::string nm = "es_mod" + std::to_string(m);
        lr = nvJitLinkAddData(h, NVJITLINK_INPUT_CUBIN, objs[m].data(), objs[m].size(), nm.c_str());
    }
    const double tc = now_ms();
    if (lr == NVJITLINK_SUCCESS) lr = nvJitLinkComplete(h);
    if (getenv("ES_VERBOSE")) fprintf(stderr, "[es] split link: create+add %.1f ms, complete %.1f ms\n", tc - tl, now_ms() - tc);
    if (lr != NVJITLINK_SUCCESS) {
        size_t n = 0;
        nvJitLinkGetErrorLogSize(h, &n);
        std::string log(n, '\0');
        if (n) nvJitLinkGetErrorLog(h, &log[0]);
        *err = "nvJitLink failed (" + std::to_string((int)lr) + "): " + log;
        nvJitLinkDestroy(&h);
        return ES_E_CUDA;
    }
    size_t n = 0;
    nvJitLinkGetLinkedCubinSize(h, &n);
    cubin->resize(n);
    nvJitLinkGetLinkedCubin(h, cubin->data());
    nvJitLinkDestroy(&h);
    if (getenv("ES_VERBOSE")) fprintf(stderr, "[es] split link: %.1f ms\n", now_ms() - tl);
    *info = "ptxas info    : Used " + std::to_string(regs) + " registers, split build of " +
            std::to_string(phases.size()) + " phases, " + std::to_string(spill) + " bytes spill stores, 0 bytes spill loads\n";
    return ES_OK;
}

thread_local bool t_batch_jit = false;

int jit_get(const LutNet &net, int threads, JitKernel **out, double *jit_ms, std::string *err,
            int opt, int parts) {
    if (opt == kJitDirect) {  // direct SASS (es_sass.cpp): no ptxas
        auto t0 = now_ms();
        std::vector<char> cubin;
        SassStats ss;
        std::string e2;
        if (sass_direct_cubin(net, threads, &cubin, &ss, &e2)) {
            const std::string img(cubin.begin(), cubin.end());
            const uint64_t key = fnv1a(img) ^ 0xD1EC7ull << 40 ^ (uint64_t)(uint32_t)threads;
            const uint64_t h2 = second_hash(img);
            {
                std::lock_guard<std::mutex> lk(g_jit_mu);
                auto it = g_cache.find(key);
                if (it != g_cache.end() && it->second->ptx_h2 == h2 && it->second->ptx_len == img.size()) {
                    *out = it->second;
                    *jit_ms = 0.0;
                    return ES_OK;
                }
            }
            JitKernel *k = new JitKernel();
            k->threads = threads;
            k->block = threads;
            k->opt = kJitDirect;
            k->parts = 1;
            k->ptx_h2 = h2;
            k->ptx_len = img.size();
            cudaError_t e = cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
            if (e == cudaSuccess) e = cudaLibraryGetKernel(&k->kernel, k->lib, "es_k1");
            if (e != cudaSuccess) {
                *err = std::string("direct SASS load: ") + cudaGetErrorString(e);
                if (k->lib) cudaLibraryUnload(k->lib);
                delete k;
                return ES_E_CUDA;
            }
            cudaFuncAttributes fa{};
            if (cudaFuncGetAttributes(&fa, (const void *)k->kernel) == cudaSuccess) k->regs = fa.numRegs;
            *jit_ms = now_ms() - t0;
            k->jit_ms = *jit_ms;
            if (getenv("ES_VERBOSE"))
                fprintf(stderr, "[es] direct SASS: %d instrs (%d LOP3, %d IMAD), %d regs, %.2f ms\n", ss.instrs, ss.lop3,
                        ss.imad, ss.regs_peak, *jit_ms);
            std::lock_guard<std::mutex> lk(g_jit_mu);
            auto it = g_cache.find(key);
            if (it != g_cache.end()) g_uncached.push_back(k);
            else g_cache[key] = k;
            *out = k;
            return ES_OK;
        }
        // no template for this variant, or the body does not fit one: the
        // split build (a cold single run) or the one-body -O1 build (a batch,
        // whose jobs already compile on parallel threads)
        if (getenv("ES_VERBOSE"))
            fprintf(stderr, "[es] direct SASS not possible (%s, peak live %d): ptxas build\n", e2.c_str(), net.peak_live);
        const int P = t_batch_jit ? 1 : (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
        opt = P >= 2 ? -P : 1;
        parts = P >= 2 ? P : 1;
    }
    std::string ptx;
    std::string skel;
    std::vector<std::string> phases;
    int region = 0;
    if (opt < 0) parts = -opt;  // build level -P: split into P phases at ptxas -O1
    // a program too small to cut, or whose slot file would not fit shared
    // memory, gets the one-body build at -O1 instead
    if (parts > 1 && (!splice_split(net, threads, parts, &skel, &phases, err, &region) || region > 200 * 1024)) {
        parts = 1;
        opt = 1;
        region = 0;
        err->clear();
    }
    if (parts > 1) {
        ptx = skel;  // the cache key covers every module
        for (const std::string &ph : phases) { ptx += "\n// ES_PHASE\n"; ptx += ph; }
    } else {
        parts = 1;
        if (!splice_body(net, threads, &ptx, err, &region)) return ES_E_BAD_PROGRAM;
    }
    const int level = parts > 1 ? -parts : effective_opt(opt);  // what the kernel is cached as
    opt = parts > 1 ? effective_opt(1) : level;                  // the ptxas level
    const uint64_t key = fnv1a(ptx) ^ (uint64_t)(uint32_t)threads ^ ((uint64_t)(opt & 7) << 56) ^
                         ((uint64_t)parts << 48);
    // the 64-bit key alone could collide: a hit must also match a second,
    // independent hash and the length of the PTX
    const uint64_t h2 = second_hash(ptx);
    auto same = [&](const JitKernel *k) { return k->ptx_h2 == h2 && k->ptx_len == ptx.size(); };
    {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end() && same(it->second)) { *out = it->second; *jit_ms = 0.0; return ES_OK; }
    }
    // compile outside the lock: batches JIT many programs on parallel threads
    NvtxRange nvtx("es_jit");
    auto t0 = now_ms();
    std::vector<char> cubin;
    std::string info;
    static const std::string version = ptxc_version();
    const uint64_t dkey = key ^ fnv1a(version) * 31u;
    const std::string dir = disk_cache_dir();
    if (!disk_load(dir, dkey, ptx, &cubin, &info)) {
        int rc = parts > 1 ? split_to_cubin(skel, phases, &cubin, &info, err, opt)
                           : ptx_to_cubin(ptx, &cubin, &info, err, opt);
        if (rc != ES_OK) return rc;
        disk_store(dir, dkey, ptx, cubin, info);
    }
    JitKernel *k = new JitKernel();
    k->threads = threads;
    k->block = threads;
    k->region_bytes = region;
    k->opt = level;
    k->parts = parts;
    k->ptx_h2 = h2;
    k->ptx_len = ptx.size();
    parse_ptxas_info(info, &k->regs, &k->spill_bytes);
    cudaError_t e = cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr,
                                        nullptr, 0);
    if (e != cudaSuccess) {
        *err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
        delete k;
        return ES_E_CUDA;
    }
    e = cudaLibraryGetKernel(&k->kernel, k->lib,
                             "es_k1");
    if (e != cudaSuccess) {
        *err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
        cudaLibraryUnload(k->lib);
        delete k;
        return ES_E_CUDA;
    }
    if (parts > 1) {  // the linked kernel's register count (the phases' ABI calls included)
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, (const void *)k->kernel) == cudaSuccess) k->regs = fa.numRegs;
    }
    *jit_ms = now_ms() - t0;
    k->jit_ms = *jit_ms;
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end() && same(it->second)) {  // another thread won the race: keep its module
        cudaLibraryUnload(k->lib);
        delete k;
        *out = it->second;
        return ES_OK;
    }
    if (it != g_cache.end()) g_uncached.push_back(k);  // key collision: keep the resident entry
    else g_cache[key] = k;
    *out = k;
    return ES_OK;
}

void jit_clear() {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    for (auto &kv : g_cache) {
        cudaLibraryUnload(kv.second->lib);
        delete kv.second;
    }
    g_cache.clear();
    for (JitKernel *k : g_uncached) {
        cudaLibraryUnload(k->lib);
        delete k;
    }
    g_uncached.clear();
}

}  // namespace es
