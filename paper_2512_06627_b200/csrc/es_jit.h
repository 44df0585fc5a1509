// es_jit.h -- K1 JIT (internal).
#pragma once

#include <chrono>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "es_core.h"

namespace es {

// Build level of a direct-SASS kernel (es_sass.cpp): below every ptxas level
// (a request for it is met by any compiled kernel, and a ptxas build of the
// same program later replaces it -- tier-up).
constexpr int kJitDirect = -1000;
// Whether a direct-SASS template exists for this K1 variant.
bool sass_template_exists(int threads, bool multi);

struct JitKernel {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    int threads = 0;        // variant selector (see below)
    int block = 0;          // CTA size of the launch
    int region_bytes = 0;   // dynamic shared memory of the launch (split build: its slot file)
    int parts = 1;          // phases of a split build (1: one straight-line body)
    int regs = -1;
    int spill_bytes = 0;
    int opt = 3;            // build level: ptxas -O3 / -O1, or -P = split build of P phases at -O1
                            // (ordered: a request for level L is met by a kernel of level >= L)
    double jit_ms = 0;
    uint64_t ptx_h2 = 0;    // second hash + length of the PTX: cache-hit check
    size_t ptx_len = 0;
};

inline double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// The complete PTX for `net` at a block size of 128/256/512 threads.
bool splice_body(const LutNet &net, int threads, std::string *ptx, std::string *err,
                 int *region_bytes = nullptr);
// PTX -> sm_100a cubin in process at ptxas -O<opt> (ES_PTXAS_O overrides);
// `info` receives ptxas's verbose log.
int ptx_to_cubin(const std::string &ptx, std::vector<char> *cubin, std::string *info,
                 std::string *err, int opt = 3, bool relocatable = false);
// Split build (es_split.cpp): the skeleton calling `parts` phase functions,
// and the phase modules; smem_bytes = the slot file per CTA.
bool splice_split(const LutNet &net, int threads, int parts, std::string *skel,
                  std::vector<std::string> *phases, std::string *err, int *smem_bytes);
int split_to_cubin(const std::string &skel, const std::vector<std::string> &phases, std::vector<char> *cubin,
                   std::string *info, std::string *err, int opt);
void parse_ptxas_info(const std::string &info, int *regs, int *spill_bytes);
// Cached compile + load at ptxas -O<opt> (1: ~40 % less compile time, a few
// % slower kernels -- for cold single runs; 3: default).  Thread-safe.
// parts > 1 (or opt = -parts): split build (cold runs: ptxas on the phases in parallel).
int jit_get(const LutNet &net, int threads, JitKernel **out, double *jit_ms, std::string *err,
            int opt = 3, int parts = 1);
void jit_clear();
// set on the threads of a batched K1 run (run_batch_jit): a failed direct-SASS
// build falls back to one ptxas body, never a split build
extern thread_local bool t_batch_jit;

// Direct-SASS K1 build (es_sass.cpp): the body lowered, scheduled, register-
// allocated and encoded by the library and patched into a placeholder skeleton
// that ptxas compiled at build time -- no ptxas at run time.  False (with
// `err`) when the variant has no template or the body does not fit it.
struct SassStats {
    int instrs = 0;      // body instructions
    int lop3 = 0, imad = 0;
    int regs_peak = 0;   // simultaneously allocated registers
    int cycles = 0;      // issue cycles of one iteration, one warp alone (model)
    int reg_lo = 0, reg_hi = 0, reg_o0 = 0, reg_o1 = 0;  // the template's interface registers
};
bool sass_direct_cubin(const LutNet &net, int threads, std::vector<char> *cubin, SassStats *st, std::string *err);
// K4 (k4_skeleton.cu): one job's body for the multi-body skeleton (encoded
// (lo, hi) words, position-independent), and a module of bodies behind the
// skeleton's indirect branch (body i = jump-table entry i)
// Template variants differ in CTAs per SM (k4_blocks: 1 = ~230 body
// registers, 2 = ~90); k4_body with variant < 0 picks the most-CTA variant
// the body's registers fit and returns it in *used.
int k4_variants();
int k4_blocks(int variant);
bool k4_body(const LutNet &net, int variant, std::vector<uint64_t> *words, SassStats *st, int *used,
             std::string *err);
bool k4_module(const std::vector<const std::vector<uint64_t> *> &bodies, int variant, std::vector<char> *cubin,
               std::vector<uint32_t> *entry, std::string *err);
int k4_body_capacity(int variant);  // instruction slots of one module
int k4_max_bodies(int variant);     // bodies per module

}  // namespace es
