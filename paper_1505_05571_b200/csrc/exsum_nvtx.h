// exsum_nvtx.h — NVTX ranges around the C-ABI entry points (header-only NVTX v3:
// a few nanoseconds when no tool is attached; named ranges in Nsight / ncu
// --nvtx when one is).
#ifndef EXSUM_NVTX_H_
#define EXSUM_NVTX_H_

#include <nvtx3/nvToolsExt.h>

namespace exsum_b200 {
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace exsum_b200

#define EXSUM_NVTX_CAT2(a, b) a##b
#define EXSUM_NVTX_CAT(a, b) EXSUM_NVTX_CAT2(a, b)
#define EXSUM_NVTX(name) ::exsum_b200::NvtxRange EXSUM_NVTX_CAT(exsum_nvtx_, __LINE__)(name)

#endif  // EXSUM_NVTX_H_
