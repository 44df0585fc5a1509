// es_jit.h -- K1 JIT (internal).
#pragma once

#include <chrono>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "es_core.h"

namespace es {

struct JitKernel {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    int threads = 0;        // variant selector (see below)
    int block = 0;          // CTA size of the launch
    int region_bytes = 0;   // (unused: 0)
    int regs = -1;
    int spill_bytes = 0;
    int opt = 3;            // ptxas optimisation level it was compiled at
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
                 std::string *err, int opt = 3);
void parse_ptxas_info(const std::string &info, int *regs, int *spill_bytes);
// Cached compile + load at ptxas -O<opt> (1: ~40 % less compile time, a few
// % slower kernels -- for cold single runs; 3: default).  Thread-safe.
int jit_get(const LutNet &net, int threads, JitKernel **out, double *jit_ms, std::string *err,
            int opt = 3);
void jit_clear();

}  // namespace es
