// Standalone block entry points of the serving path, for callers that
// hold their own K / V blocks instead of a kvlc_cache (e.g. an inference engine's
// paged cache, or the QKV-projection epilogue):
//   kvlc_quantize_pack       quantize_tensor on bf16 (K1 on a key chunk, any axis / bits / G)
//   kvlc_fwht_quantize_pack  rotate(x, H, "post") + token-wise quantize_tensor (K2)
//   kvlc_state_update        S += sum_i v_q[i] (x) phi_k(k_err[i]), P += sum_i phi_k(k_err[i]) (K3)
//   kvlc_flush_due           flush_group on every sequence the host marks due (K8 without append)
// Code decisions, scales and zeros follow the reference's float64 arithmetic
// (quantize.py:189-209), so codes are bit-identical to quantize_tensor on the same
// bf16 values; fp16 scale / zero are float16(reference float64 value).
#include <algorithm>

#include "kvlc_common.cuh"

namespace kvlc {
namespace {

__device__ __forceinline__ double load_val(const uint16_t* x, int64_t i) {
  return (double)__uint_as_float((uint32_t)x[i] << 16);
}
__device__ __forceinline__ double load_val(const double* x, int64_t i) { return x[i]; }

enum AuxMode { AUX_NONE = 0, AUX_ERR = 1, AUX_DEQ = 2 };

// _quantize_rows (quantize.py:189-209) + pack_codes (:71-94), one warp per
// (line, group); line = row (token axis) or column (channel axis, :233-237).
// Words wholly inside one group are stored; words shared by two groups (G not a
// multiple of the lane count) are OR-ed into a zeroed buffer.
// aux: AUX_ERR -> x - x_hat (k_err, cache.py:153); AUX_DEQ -> x_hat (v_q, :154),
// x_hat = code * scale + zero in float64 (quantize.py:212-217), rounded to fp32.
template <typename In>
__global__ void qpack_kernel(const In* __restrict__ x, int64_t rows, int64_t cols, int64_t ld, int axis,
                             int group, int top, int lb, int lanes, uint32_t* __restrict__ words,
                             uint16_t* __restrict__ s16, uint16_t* __restrict__ z16, float* __restrict__ aux,
                             int aux_mode, int64_t aux_ld) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool tok = axis == KVLC_AXIS_TOKEN;
  const int64_t lines = tok ? rows : cols, span = tok ? cols : rows;
  const int64_t ngroups = (span + group - 1) / group, nw = (span + lanes - 1) / lanes;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < lines * ngroups; i += nwarps) {
    const int64_t line = i / ngroups, gi = i % ngroups;
    const int64_t lo = gi * group, hi = min(span, lo + group);
    auto at = [&](int64_t j) { return tok ? line * ld + j : j * ld + line; };
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t j = lo + lane; j < hi; j += 32) {
      const double v = load_val(x, at(j));
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    mn = warp_min_d(mn);
    mx = warp_max_d(mx);
    const double scale = __ddiv_rn(__dsub_rn(mx, mn), (double)top);
    const int64_t mi = tok ? line * ngroups + gi : gi * lines + line;
    if (lane == 0) {
      s16[mi] = __half_as_ushort(__double2half(scale));
      z16[mi] = __half_as_ushort(__double2half(mn));
    }
    for (int64_t w = lo / lanes + lane; w <= (hi - 1) / lanes; w += 32) {
      const int64_t e0 = max(lo, w * lanes), e1 = min(hi, (w + 1) * lanes);
      uint32_t part = 0;
      for (int64_t j = e0; j < e1; ++j) {
        const double v = load_val(x, at(j));
        const uint32_t code = code_of(v, mn, scale, top);
        part |= code << (lb * (int)(j - w * lanes));
        if (aux_mode != AUX_NONE) {
          const double xh = __dadd_rn(__dmul_rn((double)code, scale), mn);
          aux[tok ? line * aux_ld + j : j * aux_ld + line] = (float)(aux_mode == AUX_ERR ? __dsub_rn(v, xh) : xh);
        }
      }
      uint32_t* dst = tok ? words + line * nw + w : words + w * lines + line;
      if (e0 == w * lanes && e1 == min(span, (w + 1) * lanes)) *dst = part;
      else atomicOr(dst, part);
    }
  }
}

// rotate(x, H, "post") (hadamard.py:45-57) of bf16 rows in the reference's dgemm
// order: sequential float64 FMA over the inner index from 0.0 (the same evaluation
// as kvlc_ref_rotate), H[j][c] = (-1)^popcount(j & c) / sqrt(dim).
__global__ void rotate_bf16_kernel(const uint16_t* __restrict__ x, int64_t rows, int dim, int64_t ld,
                                   double* __restrict__ out) {
  const double h = 1.0 / sqrt((double)dim);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dim;
    const int c = (int)(i % dim);
    double acc = 0.0;
    for (int j = 0; j < dim; ++j)
      acc = fma(load_val(x, r * ld + j), (__popc((unsigned)(j & c)) & 1) ? -h : h, acc);
    out[i] = acc;
  }
}

// phi_k (adapter.py:80-96) of fp32 k_err rows in float64: one block per row, logits
// x @ W1 / x @ W2 by sequential FMA, each half a max-shifted softmax (linalg.py:38-47).
__global__ void phi_rows_kernel(const float* __restrict__ x, int64_t n, int d, const float* __restrict__ w1,
                                const float* __restrict__ w2, int h, double* __restrict__ phi) {
  extern __shared__ double sh[];  // [2h] logits, [34] reduction
  double* red = sh + 2 * h;
  const int nwarp = blockDim.x >> 5, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const float* xr = x + row * d;
    for (int f = threadIdx.x; f < 2 * h; f += blockDim.x) {
      const float* w = f < h ? w1 : w2;
      const int col = f < h ? f : f - h;
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc = fma((double)xr[c], (double)w[(int64_t)c * h + col], acc);
      sh[f] = acc;
    }
    __syncthreads();
    for (int half = 0; half < 2; ++half) {
      double* s = sh + half * h;
      double m = -INFINITY;
      for (int f = threadIdx.x; f < h; f += blockDim.x) m = fmax(m, s[f]);
      m = warp_max_d(m);
      if (lane == 0) red[warp] = m;
      __syncthreads();
      m = red[0];
      for (int w = 1; w < nwarp; ++w) m = fmax(m, red[w]);
      double sum = 0.0;
      for (int f = threadIdx.x; f < h; f += blockDim.x) sum += (s[f] = exp(s[f] - m));
      sum = warp_sum_d(sum);
      __syncthreads();
      if (lane == 0) red[warp] = sum;
      __syncthreads();
      double tot = 0.0;
      for (int w = 0; w < nwarp; ++w) tot += red[w];
      for (int f = threadIdx.x; f < h; f += blockDim.x) phi[row * 2 * h + half * h + f] = s[f] / tot;
      __syncthreads();
    }
  }
}

// cache.py:155-158 over n tokens in order: each S / P element accumulates its
// float64 sum of products token by token, then adds it to the fp32 state once.
__global__ void state_add_kernel(const float* __restrict__ vq, const double* __restrict__ phi, int64_t n,
                                 int d, int rank, float* __restrict__ S, float* __restrict__ P) {
  const int64_t total = (int64_t)d * rank + rank;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (i < (int64_t)d * rank) {
      const int c = (int)(i / rank), f = (int)(i % rank);
      for (int64_t t = 0; t < n; ++t) acc = fma((double)vq[t * d + c], phi[t * rank + f], acc);
      S[i] = (float)((double)S[i] + acc);
    } else {
      const int f = (int)(i - (int64_t)d * rank);
      for (int64_t t = 0; t < n; ++t) acc += phi[t * rank + f];
      P[f] = (float)((double)P[f] + acc);
    }
  }
}

inline int grid_for(int64_t threads) {
  const int64_t b = (threads + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 64 ? 148 * 64 : b));
}

int launch_qpack_bf16(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld, int axis, int bits, int group,
                      uint32_t* words, uint16_t* s16, uint16_t* z16, float* aux, int mode, cudaStream_t s) {
  const int lanes = lanes_per_word(bits);
  const int64_t span = axis == KVLC_AXIS_TOKEN ? cols : rows, lines = axis == KVLC_AXIS_TOKEN ? rows : cols;
  if (group % lanes != 0) KVLC_CUDA(cudaMemsetAsync(words, 0, (size_t)lines * cdiv(span, lanes) * 4, s));
  qpack_kernel<uint16_t><<<grid_for(lines * cdiv(span, group) * 32), 256, 0, s>>>(
      x, rows, cols, ld, axis, group, (1 << bits) - 1, lane_bits(bits), lanes, words, s16, z16, aux, mode, cols);
  return check_launch("quantize_pack");
}

}  // namespace
}  // namespace kvlc

using namespace kvlc;

extern "C" {

int kvlc_quantize_pack(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld, int axis, int bits,
                       int group, uint32_t* words, uint16_t* scale, uint16_t* zero, float* err_opt,
                       void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(bits != 16, "bits=16 is a passthrough config; nothing to quantize");
  KVLC_REQUIRE(valid_bits(bits), "bits must be one of (2, 3, 4, 8), got %d", bits);
  KVLC_REQUIRE(group >= 1, "group_size must be >= 1, got %d", group);
  KVLC_REQUIRE(rows > 0 && cols > 0, "expected a non-empty matrix, got shape (%lld, %lld)", (long long)rows,
               (long long)cols);
  KVLC_REQUIRE(ld >= cols, "row stride %lld < cols %lld", (long long)ld, (long long)cols);
  KVLC_REQUIRE(axis == KVLC_AXIS_TOKEN || axis == KVLC_AXIS_CHANNEL, "axis must be token or channel");
  return launch_qpack_bf16(x, rows, cols, ld, axis, bits, group, words, scale, zero, err_opt,
                           err_opt ? AUX_ERR : AUX_NONE, as_stream(stream));
}

size_t kvlc_fwht_quantize_workspace(int64_t rows, int dim) { return align_up((size_t)rows * dim * sizeof(double)); }

int kvlc_fwht_quantize_pack(const uint16_t* x, int64_t rows, int dim, int64_t ld, int bits, int group,
                            uint32_t* words, uint16_t* scale, uint16_t* zero, float* vq_opt, void* ws,
                            size_t ws_bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(valid_bits(bits), "bits must be one of (2, 3, 4, 8), got %d", bits);
  KVLC_REQUIRE(group >= 1, "group_size must be >= 1, got %d", group);
  KVLC_REQUIRE(pow2(dim) && dim <= 4096, "Hadamard dimension must be a power of two, got %d", dim);
  KVLC_REQUIRE(rows > 0, "expected a non-empty matrix, got shape (%lld, %d)", (long long)rows, dim);
  KVLC_REQUIRE(ld >= dim, "row stride %lld < dim %d", (long long)ld, dim);
  KVLC_REQUIRE(ws && ws_bytes >= kvlc_fwht_quantize_workspace(rows, dim), "workspace too small (%zu bytes)",
               ws_bytes);
  cudaStream_t s = as_stream(stream);
  double* rot = static_cast<double*>(ws);
  rotate_bf16_kernel<<<grid_for(rows * dim), 256, 0, s>>>(x, rows, dim, ld, rot);
  int rc = check_launch("fwht");
  if (rc) return rc;
  const int lanes = lanes_per_word(bits);
  if (group % lanes != 0) KVLC_CUDA(cudaMemsetAsync(words, 0, (size_t)rows * cdiv(dim, lanes) * 4, s));
  qpack_kernel<double><<<grid_for(rows * cdiv(dim, group) * 32), 256, 0, s>>>(
      rot, rows, dim, dim, KVLC_AXIS_TOKEN, group, (1 << bits) - 1, lane_bits(bits), lanes, words, scale, zero,
      vq_opt, vq_opt ? AUX_DEQ : AUX_NONE, dim);
  return check_launch("fwht_quantize_pack");
}

size_t kvlc_state_update_workspace(int64_t n, int rank) { return align_up((size_t)n * rank * sizeof(double)); }

int kvlc_state_update(const float* k_err, const float* vq_rot, int64_t n, int d, int rank, const float* w1k,
                      const float* w2k, float* S, float* P, void* ws, size_t ws_bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(d >= 1 && rank >= 2 && rank % 2 == 0, "adapter dim mismatch: d=%d rank=%d", d, rank);
  KVLC_REQUIRE(k_err && vq_rot && w1k && w2k && S && P, "null argument");
  if (n <= 0) return KVLC_OK;
  KVLC_REQUIRE(ws && ws_bytes >= kvlc_state_update_workspace(n, rank), "workspace too small (%zu bytes)",
               ws_bytes);
  cudaStream_t s = as_stream(stream);
  double* phi = static_cast<double*>(ws);
  const int h = rank / 2;
  const size_t shm = (size_t)(2 * h + 34) * sizeof(double);
  KVLC_REQUIRE(shm <= 200 * 1024, "rank %d too large", rank);
  if (shm > 48 * 1024) KVLC_CUDA(cudaFuncSetAttribute(phi_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  phi_rows_kernel<<<(int)std::min<int64_t>(n, 148 * 8), 256, shm, s>>>(k_err, n, d, w1k, w2k, h, phi);
  int rc = check_launch("state_update_phi");
  if (rc) return rc;
  state_add_kernel<<<grid_for((int64_t)d * rank + rank), 256, 0, s>>>(vq_rot, phi, n, d, rank, S, P);
  return check_launch("state_update");
}

int kvlc_flush_due(const kvlc_cache* c, const kvlc_adapter* ad, const int32_t* flush_host, void* ws,
                   size_t ws_bytes, void* stream) {
  KVLC_REQUIRE(c != nullptr && c->B >= 1 && c->B <= 1024, "bad cache descriptor");
  int32_t none[1024] = {0};
  return kvlc_append(c, ad, nullptr, nullptr, none, flush_host, ws, ws_bytes, stream);
}

}  // extern "C"
