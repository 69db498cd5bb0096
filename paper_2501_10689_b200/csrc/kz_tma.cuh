// TMA staging of the packed rows H_eff into shared memory (north_star: "H is staged in shared memory via TMA").
//
// The complex64 rows h_bi live back to back in heff (kz_problem.row_val_ptr).  A kernel keeps every row in shared
// memory as whole 32-antenna chunk pieces (zero padded where the row's support [s, s+L) does not cover the
// chunk).  Each piece is one 1-D tensor copy (cp.async.bulk.tensor.1d, 32 elements x 8 B = 256 B) whose start
// coordinate is the element of heff that antenna chunk_start would have: element granularity, so no alignment
// constraint on row starts; coordinates before the mapped range read as zero (TMA out-of-bounds fill), and the
// pad lanes a piece pulls from the neighbouring rows are zeroed after the copies land.  Completion is tracked by
// one mbarrier per CTA (expect_tx per issuing thread, one arrival after all of them).
//
// The tensor map is encoded on the host per launch over the element range [val_lo, val_hi) the batch's rows
// occupy (kz_problem), coordinates relative to its 16-byte aligned base; batches whose range does not fit the
// signed 32-bit TMA coordinates (or whose range is unknown: val_hi = 0) keep the asynchronous-copy path.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "../../include/kaczmarz_b200.h"

namespace kz {

// host: whether the last launch on this thread staged H_eff with TMA (kz_last_tma_staging)
inline thread_local int g_last_tma = 0;

struct HeffTma {
  CUtensorMap map;  // 64-byte aligned (CUtensorMap's own alignment)
  long long base;   // heff element that coordinate 0 addresses
  int ok;           // 1: the TMA path is usable for this launch
  int _pad;
};

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}

// host: encode the 1-D map over heff[val_lo & ~1, val_hi) (complex64 as 8-byte elements, 32-element boxes)
inline void heff_tma_encode(const kz_problem& P, HeffTma* t) {
  t->ok = 0;
  t->base = 0;
  static const bool off = getenv("KZ_NO_TMA") != nullptr;  // A/B switch: the asynchronous-copy staging
  if (off || P.dtype != KZ_C64 || !P.heff || P.val_hi <= P.val_lo || P.val_lo < 0) return;
  const long long base = P.val_lo & ~1LL;
  const long long n = P.val_hi - base;
  if (n + 64 >= (1LL << 31)) return;  // coordinates are signed 32-bit
  void* addr = (char*)P.heff + base * 8;
  if (((uintptr_t)addr & 15) != 0) return;
  static const bool verbose = getenv("KZ_VERBOSE") != nullptr;
  auto fn = tma_encode_fn();
  if (!fn) {
    if (verbose) fprintf(stderr, "[kz tma] cuTensorMapEncodeTiled entry point unavailable\n");
    return;
  }
  cuuint64_t dim[1] = {(cuuint64_t)n};
  cuuint64_t stride[1] = {(cuuint64_t)n * 8};
  cuuint32_t box[1] = {32};
  cuuint32_t es[1] = {1};
  const CUresult r = fn(&t->map, CU_TENSOR_MAP_DATA_TYPE_INT64, 1, addr, dim, stride, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (verbose) fprintf(stderr, "[kz tma] encode n=%lld base=%lld -> %d\n", n, base, (int)r);
  if (r != CUDA_SUCCESS) return;
  t->base = base;
  t->ok = 1;
}

// host: called by the launchers right before a kernel launch
inline void note_tma(const HeffTma& t) { g_last_tma = t.ok; }

namespace tma {

constexpr uint32_t PIECE_BYTES = 32 * 8;  // one 32-antenna complex64 chunk piece

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
// 32 elements of heff starting at map coordinate x -> dst (16-byte aligned shared memory)
__device__ __forceinline__ void load_piece(void* dst, const CUtensorMap* map, int x, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::
          "r"(saddr(dst)),
      "l"((unsigned long long)map), "r"(x), "r"(saddr(mb))
      : "memory");
}

}  // namespace tma
}  // namespace kz
