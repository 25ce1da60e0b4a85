// Second unit set of a paired column + row filter launch (l1f_filter_pair_f32, filter_tc.cu).
#pragma once
#include <cstdint>

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
  int mode;  // 0: by the pass model, 1: one launch, 2: two launches
};

}  // namespace tcf
}  // namespace l1f
