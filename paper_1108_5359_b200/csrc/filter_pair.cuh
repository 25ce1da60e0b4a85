// Second unit set of a paired column + row filter launch (l1f_filter_pair_f32, filter_tc.cu).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace l1f {
namespace tcf {

struct Second {
  const float* X;
  int64_t ldx, n_units;
  const float* A;
  int64_t lda;
  float* Z;
  int64_t ldz;
  int32_t* iters;
  float* res;
  uint8_t* status;
  int mode;  // 0: by the pass model, 1: one launch, 2: two launches, 3: report the model's choice only
  int* plan_out = nullptr;  // mode 3: 1 if one grid would run, else 0
};

// host side: progress-notification targets of a single-set filter launch, passed explicitly by
// the overlapped calls (l1f_rowfilter_reconstruct_*, l1f_filter_with_gather_f32) down to the
// launch, and what that launch did
struct NotifyHost {
  const int64_t* rows = nullptr;    // output row of every unit (strip = row >> 7)
  unsigned* cnt = nullptr;          // per strip: + 1 per (unit, CTA of its cluster) with z written
  unsigned* resident = nullptr;     // + 1 per started CTA
  cudaEvent_t after_prologue = nullptr;  // recorded between the prologue and the main launch
  int cluster = 0, ctas = 0;        // out: cluster size, CTAs of the main launch (0: none)
};

}  // namespace tcf
}  // namespace l1f
