// Fast lockstep path (fixed-T, contiguous supports).  Placeholder: the
// generic kernel handles every case until the tuned kernel lands.
#pragma once

#include "kz_common.cuh"

namespace kz {

// returns 1 if launched, 0 if the problem is not eligible, -1 on launch failure
inline int lockstep_try_launch(const kz_problem&, int, const kz_stop&, const kz_rng&, const kz_out&, cudaStream_t,
                               int32_t*) {
  return 0;
}

}  // namespace kz
