// es_nvtx.h -- NVTX ranges around the engine's host phases (map, JIT, sweep,
// batch), so ncu / Nsight traces show where a verdict's time goes.  NVTX v3
// is header-only: no library to link, near-zero cost without a tool attached.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace es {

struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

}  // namespace es
