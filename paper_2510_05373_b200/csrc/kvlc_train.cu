// Adapter calibration step on the GPU: the trainer's inner loop
// (adapter.py:180-251: _batched_loss_and_grads + AdamState.step) as repo kernels, float64.
//
// For query positions p_b sharing one key set (keys 0..n-1, causal mask j <= p_b):
//   v = phi_k(k_err) [n][D], u = phi_q(q[p]) [b][D]            (kvlc_ref_feature_map)
//   num_bj = exp(q_b . khat_j / sqrt(d)) + u_b . v_j,  z_b = sum_j num_bj
//   loss = -(1/b) sum_bj a_bj log(num_bj / z_b)
//   g_bj = (1 - a_bj / w_bj) / z_b / b                           (pa_rows_kernel)
//   grad_u = g v, grad_v = g^T u                                 (gemm_f64_kernel)
//   dz = softmax_backward(u halves, grad_u halves), dk likewise  (softmax_bwd_kernel)
//   grads: w1_q = q_b^T dz[:, :h], w2_q = q_b^T dz[:, h:], w1_k = k_err^T dk[:, :h], ...
//   Adam with bias correction, betas (0.9, 0.999), eps 1e-8, in place (adam_kernel)
// All float64 (the reference's arithmetic); summation orders differ from numpy's, so the
// results agree to float64 rounding (tests/test_gpu_ref.py: 1e-12 on the gradients).
#include "kvlc_common.cuh"

extern "C" int kvlc_ref_feature_map(const double* x, int64_t n, int d, const double* w1, const double* w2, int h,
                                    double* out, void* stream);

namespace kvlc {
namespace {

// C[m][n] = sum_k A(m, k) B(k, n) (+ C when acc), arbitrary strides; 32 x 32 output tile
// per 256-thread CTA, 2 x 2 outputs per thread, K in slices of 32 through shared memory.
__global__ void __launch_bounds__(256) gemm_f64_kernel(int M, int N, int K, const double* __restrict__ A,
                                                       int64_t a_rs, int64_t a_cs, const double* __restrict__ B,
                                                       int64_t b_rs, int64_t b_cs, double* __restrict__ C,
                                                       int64_t c_rs, int acc) {
  __shared__ double as[32][33], bs[32][33];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
      const int r = i >> 5, cc = i & 31;
      const int m = m0 + r, ka = k0 + cc, kb = k0 + r, n = n0 + cc;
      as[r][cc] = (m < M && ka < K) ? A[m * a_rs + ka * a_cs] : 0.0;
      bs[r][cc] = (kb < K && n < N) ? B[kb * b_rs + n * b_cs] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double a0 = as[2 * ty][k], a1 = as[2 * ty + 1][k];
      const double b0 = bs[k][2 * tx], b1 = bs[k][2 * tx + 1];
      c[0][0] = fma(a0, b0, c[0][0]);
      c[0][1] = fma(a0, b1, c[0][1]);
      c[1][0] = fma(a1, b0, c[1][0]);
      c[1][1] = fma(a1, b1, c[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + 2 * ty + i, n = n0 + 2 * tx + j;
      if (m < M && n < N) C[m * c_rs + n] = acc ? C[m * c_rs + n] + c[i][j] : c[i][j];
    }
}

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  __syncthreads();
  return t;
}

// One CTA per batch row b: the corrected row, its loss term and d loss / d num.
__global__ void __launch_bounds__(256) pa_rows_kernel(const double* __restrict__ a_full, const double* __restrict__ q,
                                                      const double* __restrict__ khat, const double* __restrict__ u,
                                                      const double* __restrict__ v, const int32_t* __restrict__ pos,
                                                      int n, int d, int D, double inv_b, double* __restrict__ num,
                                                      double* __restrict__ g, double* __restrict__ loss_b) {
  __shared__ double red[8];
  extern __shared__ double qs[];  // [d] q row, [D] u row
  const int b = blockIdx.x, p = pos[b];
  const double* qr = q + (size_t)p * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) qs[i] = qr[i];
  for (int i = threadIdx.x; i < D; i += blockDim.x) qs[d + i] = u[(size_t)b * D + i];
  __syncthreads();
  const double isd = 1.0 / sqrt((double)d);
  double* nb = num + (size_t)b * n;
  double zp = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double x = 0.0;
    if (j <= p) {
      double s = 0.0, f = 0.0;
      for (int c = 0; c < d; ++c) s = fma(qs[c], khat[(size_t)j * d + c], s);
      for (int c = 0; c < D; ++c) f = fma(qs[d + c], v[(size_t)j * D + c], f);
      x = exp(s * isd) + f;
    }
    nb[j] = x;
    zp += x;
  }
  const double z = block_sum_d(zp, red);
  double lp = 0.0;
  const double* ar = a_full + (size_t)p * n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double gv = 0.0;
    if (j <= p) {
      const double w = nb[j] / z, a = ar[j];
      lp += a * log(w);
      gv = (1.0 - a / w) / z * inv_b;
    }
    g[(size_t)b * n + j] = gv;
  }
  const double l = block_sum_d(lp, red);
  if (threadIdx.x == 0) loss_b[b] = -l * inv_b;
}

// Rows of s (softmax outputs, two halves of width h): out = s * (grad - <grad, s>) per half.
__global__ void softmax_bwd_kernel(const double* __restrict__ s, const double* __restrict__ grad, int rows, int h,
                                   double* __restrict__ out) {
  const int r = blockIdx.x, half = blockIdx.y, lane = threadIdx.x;
  if (r >= rows) return;
  const double* sr = s + (size_t)r * 2 * h + half * h;
  const double* gr = grad + (size_t)r * 2 * h + half * h;
  double dot = 0.0;
  for (int i = lane; i < h; i += 32) dot = fma(gr[i], sr[i], dot);
  dot = warp_sum_d(dot);
  double* o = out + (size_t)r * 2 * h + half * h;
  for (int i = lane; i < h; i += 32) o[i] = sr[i] * (gr[i] - dot);
}

__global__ void gather_rows_kernel(const double* __restrict__ x, const int32_t* __restrict__ pos, int b, int d,
                                   double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < b * d; i += gridDim.x * blockDim.x)
    out[i] = x[(size_t)pos[i / d] * d + i % d];
}

// Adam with bias correction (adapter.py:230-251) on one weight tensor, in place.
__global__ void adam_kernel(double* __restrict__ w, double* __restrict__ m, double* __restrict__ v,
                            const double* __restrict__ g, int64_t count, double lr, double b1, double b2, double eps,
                            double c1, double c2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double mi = b1 * m[i] + (1.0 - b1) * g[i];
    const double vi = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    m[i] = mi;
    v[i] = vi;
    w[i] -= lr * (mi / c1) / (sqrt(vi / c2) + eps);
  }
}

__global__ void sum_kernel(const double* __restrict__ x, int n, double* __restrict__ out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  s = block_sum_d(s, red);
  if (threadIdx.x == 0) *out = s;
}

int gemm(cudaStream_t st, int M, int N, int K, const double* A, int64_t a_rs, int64_t a_cs, const double* B,
         int64_t b_rs, int64_t b_cs, double* C, int64_t c_rs) {
  gemm_f64_kernel<<<dim3((N + 31) / 32, (M + 31) / 32), 256, 0, st>>>(M, N, K, A, a_rs, a_cs, B, b_rs, b_cs, C, c_rs, 0);
  return check_launch("gemm_f64");
}

}  // namespace
}  // namespace kvlc

using namespace kvlc;

extern "C" {

size_t kvlc_adapter_grads_workspace(int64_t n, int b, int d, int rank) {
  const size_t D = (size_t)rank;
  return sizeof(double) * (align_up(n * D) * 3 + align_up(b * D) * 3 + align_up((size_t)b * n) * 2 +
                           align_up((size_t)b * d) + align_up(b) + 64);
}

int kvlc_adapter_grads(const double* a_full, const double* q, const double* khat, const double* kerr, int64_t n,
                       int d, const int32_t* pos, int b, const double* w1q, const double* w2q, const double* w1k,
                       const double* w2k, int rank, double* g1q, double* g2q, double* g1k, double* g2k, double* loss,
                       void* ws, size_t ws_bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(n >= 1 && d >= 1 && b >= 1 && rank >= 2 && rank % 2 == 0, "bad adapter-grad dims");
  KVLC_REQUIRE(ws && ws_bytes >= kvlc_adapter_grads_workspace(n, b, d, rank), "adapter-grad workspace too small");
  cudaStream_t st = as_stream(stream);
  const int D = rank, h = rank / 2;
  Arena ar(ws, ws_bytes);
  double* v = ar.take<double>((size_t)n * D);
  double* gv = ar.take<double>((size_t)n * D);
  double* dk = ar.take<double>((size_t)n * D);
  double* u = ar.take<double>((size_t)b * D);
  double* gu = ar.take<double>((size_t)b * D);
  double* dz = ar.take<double>((size_t)b * D);
  double* num = ar.take<double>((size_t)b * n);
  double* g = ar.take<double>((size_t)b * n);
  double* qb = ar.take<double>((size_t)b * d);
  double* lb = ar.take<double>((size_t)b);
  int rc;
  if ((rc = kvlc_ref_feature_map(kerr, n, d, w1k, w2k, h, v, stream))) return rc;        // v = phi_k(k_err)
  gather_rows_kernel<<<(b * d + 255) / 256, 256, 0, st>>>(q, pos, b, d, qb);
  if ((rc = check_launch("gather_rows"))) return rc;
  if ((rc = kvlc_ref_feature_map(qb, b, d, w1q, w2q, h, u, stream))) return rc;         // u = phi_q(q_b)
  const size_t smem = (size_t)(d + D) * sizeof(double);
  KVLC_REQUIRE(smem <= 48 * 1024, "head dim + rank too large (%d + %d)", d, D);
  pa_rows_kernel<<<b, 256, smem, st>>>(a_full, q, khat, u, v, pos, (int)n, d, D, 1.0 / b, num, g, lb);
  if ((rc = check_launch("adapter_rows"))) return rc;
  if ((rc = gemm(st, b, D, (int)n, g, n, 1, v, D, 1, gu, D))) return rc;                 // grad_u = g v
  if ((rc = gemm(st, (int)n, D, b, g, 1, n, u, D, 1, gv, D))) return rc;                 // grad_v = g^T u
  softmax_bwd_kernel<<<dim3(b, 2), 32, 0, st>>>(u, gu, b, h, dz);
  softmax_bwd_kernel<<<dim3((unsigned)n, 2), 32, 0, st>>>(v, gv, (int)n, h, dk);
  if ((rc = check_launch("softmax_bwd"))) return rc;
  if ((rc = gemm(st, d, h, b, qb, 1, d, dz, D, 1, g1q, h))) return rc;                   // q_b^T dz[:, :h]
  if ((rc = gemm(st, d, h, b, qb, 1, d, dz + h, D, 1, g2q, h))) return rc;
  if ((rc = gemm(st, d, h, (int)n, kerr, 1, d, dk, D, 1, g1k, h))) return rc;            // k_err^T dk[:, :h]
  if ((rc = gemm(st, d, h, (int)n, kerr, 1, d, dk + h, D, 1, g2k, h))) return rc;
  sum_kernel<<<1, 256, 0, st>>>(lb, b, loss);
  return check_launch("adapter_loss");
}

int kvlc_adam_step(double* w, double* m, double* v, const double* g, int64_t count, double lr, double beta1,
                   double beta2, double eps, int64_t step, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(count >= 0 && step >= 1, "bad Adam arguments");
  const double c1 = 1.0 - pow(beta1, (double)step), c2 = 1.0 - pow(beta2, (double)step);
  adam_kernel<<<(int)std::min<int64_t>((count + 255) / 256, 148 * 8), 256, 0, as_stream(stream)>>>(
      w, m, v, g, count, lr, beta1, beta2, eps, c1, c2);
  return check_launch("adam");
}

}  // extern "C"
