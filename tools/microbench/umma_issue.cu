// Issue cost of the decode kernel's 8-MMA + commit block (kvlc_tc.cuh mma8_commit_w)
// when the TMEM base is (a) read from shared memory (runtime, non-uniform to the
// compiler) vs (b) a compile-time constant, with per-iteration varying buffers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_issue umma_issue.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2510_05373_b200/csrc/kvlc_tc.cuh"

using namespace kvlc;

template <bool CONST_TB>
__global__ void issue(long long* out, int iters) {
  __shared__ __align__(1024) uint4 bs[2][256];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 512; i += blockDim.x) (&bs[0][0])[i] = make_uint4(0x3c003c00u, 0u, 0u, 0u);
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tb = CONST_TB ? 0u : tbase;
  long long t_issue = 0, t_all = 0;
  for (int it = 0; it < iters; ++it) {
    long long t0 = clock64();
    if (warp == 0) {
      tc::fence_after_sync();
      tc::mma8_commit_w(tb + 192, tb + 64u * (uint32_t)(it & 1), tc::bdesc(tc::smem_u32(bs[it & 1])), &mbar);
    }
    long long t1 = clock64();
    tc::mbar_wait(&mbar, (uint32_t)it & 1u);
    long long t2 = clock64();
    tc::fence_before_sync();
    __syncthreads();
    if (it > 0) {
      t_issue += t1 - t0;
      t_all += t2 - t0;
    }
  }
  if (tid == 0) {
    out[0] = t_issue / (iters - 1);
    out[1] = t_all / (iters - 1);
    out[2] = tbase;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  long long h[8];
  issue<false><<<148, 256>>>(d, 64);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("runtime tb: issue %lld cyc, issue+complete %lld cyc (tbase %lld) %s\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
  issue<true><<<148, 256>>>(d, 64);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("const   tb: issue %lld cyc, issue+complete %lld cyc (tbase %lld) %s\n", h[0], h[1], h[2],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
