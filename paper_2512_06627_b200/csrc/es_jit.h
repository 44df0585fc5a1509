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
    int threads = 0;
    int regs = -1;
    int spill_bytes = 0;
    double jit_ms = 0;
};

inline double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// The complete PTX for `net` at a block size of 128/256/512 threads.
bool splice_body(const LutNet &net, int threads, std::string *ptx, std::string *err);
// PTX -> sm_100a cubin in process; `info` receives ptxas's verbose log.
int ptx_to_cubin(const std::string &ptx, std::vector<char> *cubin, std::string *info,
                 std::string *err);
void parse_ptxas_info(const std::string &info, int *regs, int *spill_bytes);
// Cached compile + load.  Thread-safe.
int jit_get(const LutNet &net, int threads, JitKernel **out, double *jit_ms, std::string *err);
void jit_clear();

}  // namespace es
