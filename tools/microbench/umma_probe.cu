// Probe: tcgen05.mma kind::f16 with A from TMEM (fp16 subnormal 2-bit codes),
// B from shared memory (MN-major, no swizzle), D f32 in TMEM, commit to an
// mbarrier, tcgen05.ld readback.  Validates the layouts the decode kernel uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tm_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__global__ void probe(const uint32_t* __restrict__ acodes,  // [128 rows][64 cols] fp16x2 (A, K=128)
                      const __half* __restrict__ bmat,      // [128 k][16 n]
                      float* __restrict__ d_out,            // [128][16]
                      int nk) {                             // number of K=16 MMAs
  __shared__ __align__(1024) __half bs[128 * 16];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  // B: MN-major, no swizzle. cols 0-7 of row k at 16*k; cols 8-15 at 2048 + 16*k
  for (int i = tid; i < 128 * 16; i += 128) {
    const int k = i / 16, n = i % 16;
    bs[(n >= 8 ? 1024 : 0) + 8 * k + (n & 7)] = bmat[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tbase;
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
  // A: row = tid, 64 columns
  for (int c0 = 0; c0 < 64; c0 += 8) {
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = acodes[tid * 64 + c0 + j];
    tm_st8(tb + lane_off + c0, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t idesc = (1u << 4) | (1u << 16) | (2u << 17) | (8u << 24);
    const uint32_t d_t = tb + 128;
    for (int j = 0; j < nk; ++j) {
      const uint32_t saddr = smem_u32(bs) + j * 256;
      const uint64_t desc = (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) |
                            ((uint64_t)(2048 >> 4) << 32) | (1ull << 46);
      const uint32_t a_t = tb + 8 * j;
      const uint32_t acc = j > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_t),
          "r"(a_t), "l"(desc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        smem_u32(&mbar)));
  }
  // wait phase 0
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t r[16];
  tm_ld16(tb + lane_off + 128, r);
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  for (int n = 0; n < 16; ++n) d_out[tid * 16 + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tb), "r"(256));
}

int main() {
  srand(1);
  // A codes: per row m, K element k (channel): code c in 0..3, stored as fp16 subnormal c*4^p*2^-24
  // where p = (k >> 1) & 3 (the bit pair of the packed word); B rows carry 4^-p.
  std::vector<uint32_t> a(128 * 64);
  std::vector<int> code(128 * 128);
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < 128; ++k) code[m * 128 + k] = rand() & 3;
  for (int m = 0; m < 128; ++m)
    for (int j = 0; j < 64; ++j) {
      const int p = j & 3;
      uint32_t lo = (uint32_t)code[m * 128 + 2 * j] << (2 * p);
      uint32_t hi = (uint32_t)code[m * 128 + 2 * j + 1] << (2 * p);
      a[m * 64 + j] = lo | (hi << 16);
    }
  std::vector<__half> b(128 * 16);
  std::vector<double> bd(128 * 16);
  for (int k = 0; k < 128; ++k)
    for (int n = 0; n < 16; ++n) {
      const int p = (k >> 1) & 3;
      double v = ((rand() / (double)RAND_MAX) * 2 - 1) * 3.0;
      __half h = __float2half((float)(v / pow(4.0, p)));
      b[k * 16 + n] = h;
      bd[k * 16 + n] = (double)__half2float(h);
    }
  uint32_t* da; __half* db; float* dd;
  CK(cudaMalloc(&da, a.size() * 4)); CK(cudaMalloc(&db, b.size() * 2)); CK(cudaMalloc(&dd, 128 * 16 * 4));
  CK(cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
  probe<<<1, 128>>>(da, db, dd, 8);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> d(128 * 16);
  CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0, mx = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      double ref = 0;
      for (int k = 0; k < 128; ++k) {
        const int p = (k >> 1) & 3;
        ref += code[m * 128 + k] * pow(4.0, p) * bd[k * 16 + n];
      }
      double got = (double)d[m * 16 + n] * 16777216.0;
      worst = fmax(worst, fabs(got - ref));
      mx = fmax(mx, fabs(ref));
      if (m < 2 && n < 4) printf("m%d n%d ref %.6f got %.6f\n", m, n, ref, got);
    }
  printf("umma_probe f16 TS (A tmem subnormal, B MN-major): max abs err %.3e of max %.3e -> %s\n", worst, mx,
         worst <= 1e-5 * mx ? "PASS" : "FAIL");
  return 0;
}
