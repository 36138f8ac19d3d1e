// Probe of the legacy warp-level tensor path on sm_100a, used to choose the
// decode kernel's inner product formulation.
//   1. mma.sync throughput: f16/bf16 m16n8k16 (f32 acc), s8/u8 m16n8k32 (s32 acc)
//   2. fp16 subnormal operands: are codes stored as c * 4^j * 2^-24 exact?
//   3. movmatrix.trans layout check
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ILP = 8;

template <int KIND>
__global__ void __launch_bounds__(128) mma_tput(int iters, float* sink) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  for (int i = 0; i < 2; ++i) b[i] = 0x3c003c00u ^ (threadIdx.x * 3 + i);
  float acc[ILP][4] = {};
  int32_t iacc[ILP][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      if (KIND == 0) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 1) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 2) {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(iacc[j][0]), "+r"(iacc[j][1]), "+r"(iacc[j][2]), "+r"(iacc[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 3) {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(iacc[j][0]), "+r"(iacc[j][1]), "+r"(iacc[j][2]), "+r"(iacc[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else {
        // f16 accumulate
        uint32_t* h = reinterpret_cast<uint32_t*>(&iacc[j][0]);
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};\n"
                     : "+r"(h[0]), "+r"(h[1])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      }
    }
  }
  float s = 0.f;
  for (int j = 0; j < ILP; ++j)
    for (int i = 0; i < 4; ++i) s += acc[j][i] + (float)iacc[j][i];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

// A holds fp16 subnormals c*4^j*2^-24 (as produced by a single LOP3 mask of the
// packed 2-bit words); B holds normal fp16 values. Compare with exact products.
__global__ void subnormal_check(const uint32_t* a_in, const uint32_t* b_in, float* c_out) {
  int lane = threadIdx.x;
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = a_in[lane * 4 + i];
  for (int i = 0; i < 2; ++i) b[i] = b_in[lane * 2 + i];
  float c[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  for (int i = 0; i < 4; ++i) c_out[lane * 4 + i] = c[i];
}

__global__ void movmatrix_check(uint32_t* out) {
  int lane = threadIdx.x;
  int g = lane >> 2, t = lane & 3;
  // element (row g, col 2t / 2t+1) = row*8+col as fp16
  __half lo = __int2half_rn(g * 8 + 2 * t), hi = __int2half_rn(g * 8 + 2 * t + 1);
  __half2 h = __halves2half2(lo, hi);
  uint32_t x = *reinterpret_cast<uint32_t*>(&h), y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  out[lane] = y;
}

__global__ void copy_kernel(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

template <int KIND>
int run_tput(const char* name, double flop_per_mma) {
  float* sink;
  CK(cudaMalloc(&sink, 4096));
  int blocks = 148 * 8, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  mma_tput<KIND><<<blocks, 128>>>(64, sink);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  mma_tput<KIND><<<blocks, 128>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double mmas = (double)blocks * 4 * iters * ILP;
  printf("%-26s %8.1f TFLOP/s (or TOP/s)   %.3f ms   %.2f mma/clk/SM @1.965GHz\n", name,
         mmas * flop_per_mma / (ms * 1e-3) / 1e12, ms, mmas / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(sink);
  return 0;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sm_%d%d SMs %d\n", p.name, p.major, p.minor, p.multiProcessorCount);
  run_tput<0>("f16 m16n8k16 f32acc", 2.0 * 16 * 8 * 16);
  run_tput<1>("bf16 m16n8k16 f32acc", 2.0 * 16 * 8 * 16);
  run_tput<4>("f16 m16n8k16 f16acc", 2.0 * 16 * 8 * 16);
  run_tput<2>("s8 m16n8k32 s32acc", 2.0 * 16 * 8 * 32);
  run_tput<3>("u8s8 m16n8k32 s32acc", 2.0 * 16 * 8 * 32);

  // subnormal check: A (16x16) row r col k = code(r,k) * 4^j * 2^-24, j = r % 4
  uint32_t ha[128], hb[64];
  float ref[16][8];
  uint16_t A[16][16], B[16][8];
  float Af[16][16], Bf[16][8];
  for (int r = 0; r < 16; ++r)
    for (int k = 0; k < 16; ++k) {
      int code = (r * 5 + k * 3) & 3, j = r & 3;
      uint16_t bits = (uint16_t)(code << (2 * j));
      A[r][k] = bits;
      Af[r][k] = (float)code * (float)(1 << (2 * j)) * 5.9604644775390625e-8f;
    }
  for (int k = 0; k < 16; ++k)
    for (int n = 0; n < 8; ++n) {
      float v = (float)((k * 13 + n * 7) % 29 - 14) * 1037.25f;
      __half h = __float2half_rn(v);
      B[k][n] = *reinterpret_cast<uint16_t*>(&h);
      Bf[k][n] = __half2float(h);
    }
  for (int r = 0; r < 16; ++r)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += (double)Af[r][k] * Bf[k][n];
      ref[r][n] = (float)s;
    }
  for (int lane = 0; lane < 32; ++lane) {
    int g = lane >> 2, t = lane & 3;
    auto pk = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
    ha[lane * 4 + 0] = pk(A[g][2 * t], A[g][2 * t + 1]);
    ha[lane * 4 + 1] = pk(A[g + 8][2 * t], A[g + 8][2 * t + 1]);
    ha[lane * 4 + 2] = pk(A[g][2 * t + 8], A[g][2 * t + 9]);
    ha[lane * 4 + 3] = pk(A[g + 8][2 * t + 8], A[g + 8][2 * t + 9]);
    hb[lane * 2 + 0] = pk(B[2 * t][g], B[2 * t + 1][g]);
    hb[lane * 2 + 1] = pk(B[2 * t + 8][g], B[2 * t + 9][g]);
  }
  uint32_t *da, *db; float* dc;
  CK(cudaMalloc(&da, sizeof(ha))); CK(cudaMalloc(&db, sizeof(hb))); CK(cudaMalloc(&dc, 128 * 4));
  cudaMemcpy(da, ha, sizeof(ha), cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, sizeof(hb), cudaMemcpyHostToDevice);
  subnormal_check<<<1, 32>>>(da, db, dc);
  float hc[128];
  CK(cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost));
  int bad = 0; double maxrel = 0;
  for (int lane = 0; lane < 32; ++lane) {
    int g = lane >> 2, t = lane & 3;
    float got[4] = {hc[lane * 4], hc[lane * 4 + 1], hc[lane * 4 + 2], hc[lane * 4 + 3]};
    float want[4] = {ref[g][2 * t], ref[g][2 * t + 1], ref[g + 8][2 * t], ref[g + 8][2 * t + 1]};
    for (int i = 0; i < 4; ++i) {
      double rel = fabs((double)got[i] - want[i]) / (fabs((double)want[i]) + 1e-30);
      if (rel > maxrel) maxrel = rel;
      if (got[i] != want[i]) ++bad;
    }
  }
  printf("fp16 subnormal A operands: %d/128 inexact, max rel err %.3e (0 => subnormals honoured)\n", bad, maxrel);

  uint32_t* dm; CK(cudaMalloc(&dm, 32 * 4));
  movmatrix_check<<<1, 32>>>(dm);
  uint32_t hm[32]; CK(cudaMemcpy(hm, dm, sizeof(hm), cudaMemcpyDeviceToHost));
  int mbad = 0;
  for (int lane = 0; lane < 32; ++lane) {
    int g = lane >> 2, t = lane & 3;
    __half2 h = *reinterpret_cast<__half2*>(&hm[lane]);
    // transposed: thread (g,t) holds row g of M^T = column g of M, entries rows 2t,2t+1
    int lo = (int)__low2float(h), hi = (int)__high2float(h);
    if (lo != (2 * t) * 8 + g || hi != (2 * t + 1) * 8 + g) ++mbad;
  }
  printf("movmatrix.trans layout: %d/32 lanes wrong\n", mbad);

  size_t bytes = 1ull << 31;
  int4 *x, *y;
  CK(cudaMalloc(&x, bytes)); CK(cudaMalloc(&y, bytes));
  cudaMemset(x, 1, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<148 * 16, 256>>>(x, y, bytes / 16);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("copy kernel: %.1f GB/s (read+write)\n", 2.0 * bytes / (best * 1e-3) / 1e9);
  return 0;
}
