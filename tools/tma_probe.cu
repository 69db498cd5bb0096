// Probe of the TMA staging pattern used by csrc/kz_tma.cuh: a 1-D tensor map over complex64 elements (8 B), 32-
// element boxes at arbitrary (odd, negative) coordinates into 128-byte aligned shared memory, completion through
// one mbarrier (expect_tx per issuing thread, one arrival), in a plain launch and in a 2-CTA cluster launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -o tools/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2501_10689_b200/csrc/kz_tma.cuh"

struct Args {
  kz::HeffTma tma;
  const long long* coords;
  long long* out;
  int npieces;
  int kind;
  const CUtensorMap* gmap;  // kind 3: the map in global memory
  const long long* src;     // kind 4: plain bulk copies (16-byte aligned coordinates)
};

// MODE 0: expect_tx per issuing thread + one arrival (kz_tma.cuh); 1: one arrive.expect_tx of the total by
// thread 0, then the copies; 2: as 1 without the mbarrier_init fence; 3: as 1, single-thread issue
template <int MODE>
__global__ void __launch_bounds__(128) probe(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* mbar = (uint64_t*)sm;
  long long* buf = (long long*)(sm + 128);
  const uint32_t mb = kz::tma::saddr(mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(1) : "memory");
    if (MODE != 2) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (MODE == 0) {
    for (int p = threadIdx.x; p < a.npieces; p += blockDim.x) {
      kz::tma::mbar_expect(mbar, kz::tma::PIECE_BYTES);
      kz::tma::load_piece(buf + 32 * p, &a.tma.map, (int)a.coords[p], mbar);
    }
    __syncthreads();
    if (threadIdx.x == 0) kz::tma::mbar_arrive(mbar);
  } else {
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                   "r"(kz::tma::PIECE_BYTES * a.npieces) : "memory");
    __syncthreads();
    if (MODE != 3 || threadIdx.x == 0)
      for (int p = MODE == 3 ? 0 : threadIdx.x; p < a.npieces; p += MODE == 3 ? 1 : blockDim.x)
        if (a.kind == 2)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                  "r"(kz::tma::saddr(buf + 32 * p)), "l"((unsigned long long)&a.tma.map), "r"((int)a.coords[p]), "r"(0),
              "r"(mb) : "memory");
        else if (a.kind == 4)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                           "r"(kz::tma::saddr(buf + 32 * p)), "l"(a.src + (a.coords[p] & ~1LL)), "r"(256), "r"(mb)
                       : "memory");
        else if (a.kind == 3)
          kz::tma::load_piece(buf + 32 * p, a.gmap, (int)a.coords[p], mbar);
        else
          kz::tma::load_piece(buf + 32 * p, &a.tma.map, (int)a.coords[p], mbar);
  }
  kz::tma::mbar_wait(mbar, 0);
  for (int e = threadIdx.x; e < 32 * a.npieces; e += blockDim.x)
    a.out[(size_t)blockIdx.x * 32 * a.npieces + e] = buf[e];
}

int main(int argc, char** argv) {
  const long long n = 100004;
  std::vector<long long> h(n);
  for (long long i = 0; i < n; ++i) h[i] = i * 7 + 1;
  long long* d;
  cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  const int np = 37;
  std::vector<long long> co(np);
  for (int p = 0; p < np; ++p) co[p] = (p * 2711 + 13) % (n - 40) - (p == 0 ? 20 : 0);
  long long *dc, *dout;
  cudaMalloc(&dc, np * 8);
  cudaMalloc(&dout, 2 * 32 * np * 8);
  cudaMemcpy(dc, co.data(), np * 8, cudaMemcpyHostToDevice);
  kz_problem P{};
  P.dtype = KZ_C64;
  P.heff = d;
  P.val_lo = 0;
  P.val_hi = n;
  Args a{};
  kz::heff_tma_encode(P, &a.tma);
  const int kind = argc > 3 ? atoi(argv[3]) : 0;  // 0: kz_tma (1-D INT64); 1: 1-D FLOAT32; 2: 2-D FLOAT32
  if (kind == 3) {
    CUtensorMap* g;
    cudaMalloc(&g, sizeof(CUtensorMap));
    cudaMemcpy(g, &a.tma.map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    a.gmap = g;
  } else if (kind) {
    auto fn = kz::tma_encode_fn();
    cuuint64_t dim[2] = {(cuuint64_t)n, 1};
    cuuint64_t st[1] = {(cuuint64_t)(n * 8)};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(&a.tma.map, CU_TENSOR_MAP_DATA_TYPE_INT64, kind == 1 ? 1 : 2, d, dim, st, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode kind %d -> %d\n", kind, (int)r);
  }
  printf("encode ok %d\n", a.tma.ok);
  a.coords = dc;
  a.out = dout;
  a.npieces = np;
  a.kind = kind;
  a.src = d;
  const size_t smem = 128 + 32 * np * 8;
  void (*kerns[4])(Args) = {probe<0>, probe<1>, probe<2>, probe<3>};
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const bool nonneg = argc > 2 && atoi(argv[2]);
  if (nonneg) {
    co[0] = 5;
    cudaMemcpy(dc, co.data(), np * 8, cudaMemcpyHostToDevice);
  }
  cudaFuncSetAttribute(kerns[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  printf("mode %d nonneg %d\n", mode, (int)nonneg);
  for (int cl = 1; cl <= 2; ++cl) {
    cudaMemset(dout, 0xff, 2 * 32 * np * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kerns[mode], a);
    cudaError_t e2 = cudaDeviceSynchronize();
    std::vector<long long> out(2 * 32 * np);
    cudaMemcpy(out.data(), dout, out.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int b = 0; b < 2; ++b)
      for (int p = 0; p < np; ++p)
        for (int j = 0; j < 32; ++j) {
          const long long x = co[p] + j;
          const long long want = (x < 0 || x >= n) ? 0 : h[x];
          if (out[(size_t)b * 32 * np + 32 * p + j] != want) ++bad;
        }
    printf("cluster %d: launch %s, sync %s, mismatches %d\n", cl, cudaGetErrorString(e), cudaGetErrorString(e2), bad);
    if (e2 != cudaSuccess) return 1;
  }
  return 0;
}
