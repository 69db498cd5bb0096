// Bulk-copy (TMA engine) staging of the packed rows H_eff into shared memory.
//
// The complex64 rows h_bi live back to back in heff (kz_problem.row_val_ptr).  The on-chip kernels keep every
// row in shared memory as whole 32-antenna chunk pieces, zero padded where the row's support [s, s+L) does not
// cover a chunk; the element for antenna a of row i sits at an even shared-memory element index + (a mod 32)
// within its chunk piece, so its parity is a's.  The row's elements in heff start at row_val_ptr[i]: antenna a at
// element row_val_ptr[i] + a - s.  When that index has a's parity (row_val_ptr[i] - s even) the row's
// contiguous run of antennas, widened to even antenna bounds, is ONE cp.async.bulk copy (16-byte aligned source
// and destination, size a multiple of 16 B: the bulk-copy engine, SASS UBLKCP) completing on the CTA's mbarrier;
// the one neighbour element a widened bound may pull in lands in a pad lane and is zeroed afterwards with the
// other pads.  Rows of the other parity, and rows whose widened range would leave [val_lo, val_hi) (the batch's
// first / last row), are staged with 8-byte asynchronous copies (LDGSTS).  With dense packing about half the
// rows take each path.
//
// The tensor form (cp.async.bulk.tensor with a CUtensorMap, element-granular coordinates: every row by TMA) is
// the natural tool here; on this pool's driver (580.178, CUDA 12.9 runtime) UTMALDG raised "illegal instruction"
// even for the canonical 2-D example (tools/tma_std.cu, tools/tma_probe.cu), so it is not used.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/kaczmarz_b200.h"

namespace kz {

// host: whether the last launch on this thread staged rows with bulk copies (kz_last_tma_staging)
inline thread_local int g_last_tma = 0;

// host: bulk staging usable for this problem (value range known, 16-byte aligned heff, complex64)
inline int bulk_staging_ok(const kz_problem& P) {
  static const bool off = getenv("KZ_NO_TMA") != nullptr;  // A/B switch: asynchronous-copy staging only
  return !off && P.dtype == KZ_C64 && P.heff && P.val_hi > P.val_lo && P.val_lo >= 0 &&
                 ((uintptr_t)P.heff & 15) == 0
             ? 1
             : 0;
}
inline void note_tma(int ok) { g_last_tma = ok; }

namespace tma {

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(mb)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// add `bytes` to the barrier's expected transaction count (no arrival)
__device__ __forceinline__ void mbar_expect(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(saddr(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(saddr(mb)), "r"(parity)
        : "memory");
  } while (!done);
}
// bytes (multiple of 16) from 16-byte aligned global src to 16-byte aligned shared dst, completing on mb
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(mb))
               : "memory");
}

// One contiguous antenna run [r0, r1) (even chunk bounds) of row (s, L, rvo) whose shared-memory copy of antenna
// r0 is at dst: issue its bulk copy when the parity / bounds allow (returns true), else nothing (returns false).
__device__ __forceinline__ bool stage_run_bulk(float2* dst, const float2* heff, long long rvo, int s, int L, int r0,
                                               int r1, long long val_lo, long long val_hi, uint64_t* mb) {
  if (((rvo - s) & 1) != 0) return false;
  const int a0 = max(r0, s) & ~1, a1 = (min(r1, s + L) + 1) & ~1;  // widened to even antennas (within the run)
  if (a1 <= a0) return true;                                        // nothing of the row in this run
  const long long e0 = rvo + (a0 - s), e1 = rvo + (a1 - s);
  if (e0 < val_lo || e1 > val_hi) return false;
  const uint32_t bytes = (uint32_t)(a1 - a0) * 8u;
  mbar_expect(mb, bytes);
  bulk_copy(dst + (a0 - r0), heff + e0, bytes, mb);
  return true;
}

}  // namespace tma
}  // namespace kz
