// Latency probe for the decode pipeline's tcgen05 round trips (one CTA, 128 threads):
//   (a) tid 0 issues `nm` MMAs (kind::f16, M=128, N=16, K=16, A in TMEM) + commit,
//       all threads wait on the mbarrier  -> cycles per round trip
//   (b) STTM.x32 x2 + wait::st            -> cycles
//   (c) LDTM.x8 + wait::ld                -> cycles
//   (d) __syncthreads                     -> cycles
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_latency umma_latency.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2510_05373_b200/csrc/kvlc_tc.cuh"

using namespace kvlc;

__device__ __forceinline__ void mma_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %3, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(acc), "r"(tc::IDESC_F16_M128_N16)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(tc::smem_u32(bar)) : "memory");
}
// MODE 0: tid 0 issues; 1: warp 0 issues with elect.sync; 2: warps 0-3 each issue NM/4 (own D), commit each
template <int NM, int ND, int MODE = 0>
__global__ void lat(long long* out, int iters) {
  __shared__ __align__(1024) uint4 bs[256];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 256; i += blockDim.x) bs[i] = make_uint4(0x3c003c00u, 0u, 0u, 0u);
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  if (tid == 0) {
    tc::mbar_init(&mbar, MODE == 2 ? 4 : 1);
    tc::mbar_fence_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tb = tbase, la = tb + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t r[32];
  for (int j = 0; j < 32; ++j) r[j] = 0x00010001u * (j & 3);
  tc::tmem_st32(la, r);
  tc::tmem_st32(la + 32, r);
  tc::wait_st();
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  const uint32_t ba = tc::smem_u32(bs);
  const uint64_t d0 = tc::bdesc(ba);
  long long t_mma = 0, t_st = 0, t_ld = 0, t_bar = 0;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    long long t0 = clock64();
    if (MODE == 0) {
      if (tid == 0) {
        tc::fence_after_sync();
#pragma unroll
        for (int j = 0; j < NM; ++j) tc::mma_f16_ts(tb + 128 + 16 * (j % ND), tb + 8 * (j & 7), d0 + 16 * (j & 7), j >= ND);
        tc::mma_commit(&mbar);
      }
    } else if (MODE == 1) {
      if (warp == 0) {
        tc::fence_after_sync();
#pragma unroll
        for (int j = 0; j < NM; ++j) mma_elect(tb + 128 + 16 * (j % ND), tb + 8 * (j & 7), d0 + 16 * (j & 7), j >= ND);
        commit_elect(&mbar);
      }
    } else {
      tc::fence_after_sync();
#pragma unroll
      for (int j = 0; j < NM / 4; ++j) mma_elect(tb + 128 + 16 * warp, tb + 8 * (j & 7), d0 + 16 * (j & 7), j > 0);
      commit_elect(&mbar);
    }
    tc::mbar_wait(&mbar, (uint32_t)it & 1u);
    tc::fence_after_sync();
    long long t1 = clock64();
    tc::tmem_st32(la, r);
    tc::tmem_st32(la + 32, r);
    tc::wait_st();
    long long t2 = clock64();
    uint32_t d[8];
    tc::tmem_ld8(la + 128, d);
    tc::wait_ld();
    acc += d[0];
    long long t3 = clock64();
    tc::fence_before_sync();
    __syncthreads();
    long long t4 = clock64();
    if (it > 0) {
      t_mma += t1 - t0;
      t_st += t2 - t1;
      t_ld += t3 - t2;
      t_bar += t4 - t3;
    }
  }
  if (tid == 0) {
    out[0] = t_mma / (iters - 1);
    out[1] = t_st / (iters - 1);
    out[2] = t_ld / (iters - 1);
    out[3] = t_bar / (iters - 1);
    out[4] = acc;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tb, 256);
}

template <int NM, int ND, int MODE>
void run(long long* d, int grid) {
  lat<NM, ND, MODE><<<grid, 128>>>(d, 50);
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode=%d grid=%d nd=%d nm=%2d  mma+commit+wait %lld cyc  (%.1f cyc/mma) (%s)\n", MODE, grid, ND, NM, h[0],
         h[0] / (double)NM, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  run<16, 1, 0>(d, 1);
  run<32, 1, 0>(d, 1);
  run<16, 1, 1>(d, 1);
  run<32, 1, 1>(d, 1);
  run<32, 4, 1>(d, 1);
  run<16, 4, 2>(d, 1);
  run<32, 4, 2>(d, 1);
  run<64, 4, 2>(d, 1);
  run<32, 4, 2>(d, 296);
  run<32, 1, 1>(d, 296);
  return 0;
}
