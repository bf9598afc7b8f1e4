#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace atp {

enum EwKind : int {
  EW_GELU = 0,      // out = GeLU(a)                       [rows, cols]
  EW_DGELU = 1,     // out = out * GeLU'(a)                (in place)
  EW_ADD = 2,       // out = a + out                       (in place)
  EW_CORE_FWD = 3,  // out[rows, cols] = sum_s a[rows, 3*cols] per head
  EW_CORE_BWD = 4,  // out[rows, 3*cols] = expand(a[rows, cols])
  EW_COLSUM = 5,    // out (fp32 [cols]) = column sums of a [rows, cols]
};

struct EwDesc {
  int kind = EW_ADD;
  void* out = nullptr;
  const void* a = nullptr;
  int64_t rows = 0, cols = 0;  // cols: width of `out` (core_fwd) / of `a` (core_bwd, colsum)
  int heads = 1;
  int dtype = 0;  // 0 = bf16, 1 = fp32 (check mode)
};

constexpr int kMaxGroup = 16;
struct GroupSumArgs {
  void* buf[kMaxGroup];
  int p = 0;
};

cudaError_t ew_launch(const EwDesc& e, cudaStream_t st);
cudaError_t group_sum_launch(const GroupSumArgs& g, int64_t n, int dtype, cudaStream_t st);

}  // namespace atp
