// Reference-semantics kernels (float64, any d / G / bits / rank).
//
// These back the per-head drop-in shim (KVCacheState, quantize_tensor,
// rotate, feature_map, decode_step_blocked) for every shape the reference
// accepts.  They reproduce the reference's arithmetic order where that decides
// bits (the code decision, dequantisation, the S/P accumulation order) and
// its float32 block arithmetic in decode.  The batched serving path lives in
// kvlc_flush.cu / kvlc_decode.cu.
#include "kvlc_common.cuh"

namespace kvlc {
namespace {

constexpr int kThreads = 256;

inline int blocks_for(int64_t n, int t = kThreads) {
  int64_t b = (n + t - 1) / t;
  return (int)(b < 1 ? 1 : (b > 1048576 ? 1048576 : b));
}

// ---------------------------------------------------------------- packing --
// pack_codes (quantize.py:71-94): each row packs independently, code i of a
// word at bits [lb*i, lb*(i+1)), trailing lanes zero.
__global__ void pack_rows_kernel(const uint8_t* __restrict__ codes, int64_t rows, int64_t n,
                                 int lb, int lanes, uint32_t* __restrict__ words) {
  int64_t nw = (n + lanes - 1) / lanes;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * nw;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / nw, w = i % nw;
    uint32_t word = 0;
    for (int l = 0; l < lanes; ++l) {
      int64_t c = w * lanes + l;
      if (c < n) word |= (uint32_t)codes[r * n + c] << (lb * l);
    }
    words[i] = word;
  }
}

// Channel-axis packing: codes [rows][cols] packed down the columns into
// words [ceil(rows/L)][cols] (the transpose of pack_rows on x.T).
__global__ void pack_cols_kernel(const uint8_t* __restrict__ codes, int64_t rows, int64_t cols,
                                 int lb, int lanes, uint32_t* __restrict__ words) {
  int64_t nw = (rows + lanes - 1) / lanes;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw * cols;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = i / cols, c = i % cols;
    uint32_t word = 0;
    for (int l = 0; l < lanes; ++l) {
      int64_t r = w * lanes + l;
      if (r < rows) word |= (uint32_t)codes[r * cols + c] << (lb * l);
    }
    words[i] = word;
  }
}

// unpack_codes (quantize.py:97-114).
__global__ void unpack_kernel(const uint32_t* __restrict__ words, int64_t rows, int64_t nwords,
                              int64_t count, int lb, int lanes, uint32_t mask,
                              uint8_t* __restrict__ codes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * count;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / count, c = i % count;
    uint32_t w = words[r * nwords + c / lanes];
    codes[i] = (uint8_t)((w >> (lb * (c % lanes))) & mask);
  }
}

// ------------------------------------------------------------ quantization --
// _quantize_rows (quantize.py:189-209) over groups of one axis.  One thread
// per (line, group): min/max, fp64 scale, codes via code_of().
// axis token: line = row, group spans columns.  axis channel: line = column,
// group spans rows (quantize.py:236 transposes).
__global__ void quantize_groups_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                       int group, int top, int axis, double* __restrict__ scales,
                                       double* __restrict__ zeros, uint8_t* __restrict__ codes) {
  int64_t lines = axis == KVLC_AXIS_TOKEN ? rows : cols;
  int64_t span = axis == KVLC_AXIS_TOKEN ? cols : rows;
  int64_t ngroups = (span + group - 1) / group;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lines * ngroups;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t line = i / ngroups, gi = i % ngroups;
    int64_t lo = gi * group, hi = min(span, lo + group);
    auto at = [&](int64_t j) -> int64_t {
      return axis == KVLC_AXIS_TOKEN ? line * cols + j : j * cols + line;
    };
    double mn = x[at(lo)], mx = mn;
    for (int64_t j = lo + 1; j < hi; ++j) {
      double v = x[at(j)];
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    double scale = __ddiv_rn(__dsub_rn(mx, mn), (double)top);
    int64_t mi = axis == KVLC_AXIS_TOKEN ? line * ngroups + gi : gi * cols + line;
    scales[mi] = scale;
    zeros[mi] = mn;
    for (int64_t j = lo; j < hi; ++j) codes[at(j)] = (uint8_t)code_of(x[at(j)], mn, scale, top);
  }
}

// _dequantize_rows (quantize.py:212-217): code * scale + zero as two
// separately rounded fp64 operations (numpy evaluates codes*s, then + z).
__global__ void dequantize_kernel(const uint32_t* __restrict__ words, const double* __restrict__ scales,
                                  const double* __restrict__ zeros, int64_t rows, int64_t cols,
                                  int group, int lb, int lanes, uint32_t mask, int axis,
                                  double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * cols;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i % cols;
    uint32_t code;
    int64_t mi;
    if (axis == KVLC_AXIS_TOKEN) {
      int64_t nw = (cols + lanes - 1) / lanes;
      code = (words[r * nw + c / lanes] >> (lb * (c % lanes))) & mask;
      int64_t ng = (cols + group - 1) / group;
      mi = r * ng + c / group;
    } else {
      code = (words[(r / lanes) * cols + c] >> (lb * (r % lanes))) & mask;
      mi = (r / group) * cols + c;
    }
    out[i] = __dadd_rn(__dmul_rn((double)code, scales[mi]), zeros[mi]);
  }
}

// --------------------------------------------------------------- rotation --
// rotate (hadamard.py:45-57): x @ H (post) or H @ x (pre) with
// H[j][c] = (-1)^popcount(j & c) / sqrt(dim).  Evaluated as the reference's
// numpy/OpenBLAS dgemm does it: a sequential FMA accumulation over the inner
// index from 0.0 — bit-identical outputs, hence bit-identical codes even at
// rounding ties of the later quantization (O(dim^2) per line; the serving
// path uses an FWHT plus an exact re-evaluation of near-tie tokens instead).
__global__ void rotate_dense_kernel(const double* __restrict__ x, int64_t lines, int dim,
                                    int64_t stride_line, int64_t stride_elem, double* __restrict__ out) {
  const double h = 1.0 / sqrt((double)dim);
  const int64_t total = lines * dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = i / dim;
    const int c = (int)(i % dim);
    const double* xl = x + line * stride_line;
    double acc = 0.0;
    for (int j = 0; j < dim; ++j) {
      const double hjc = (__popc((unsigned)(j & c)) & 1) ? -h : h;
      acc = fma(xl[j * stride_elem], hjc, acc);
    }
    out[line * stride_line + c * stride_elem] = acc;
  }
}

// ------------------------------------------------------------ feature map --
// feature_map (adapter.py:80-88): one block per row; each half is a
// max-shifted softmax (linalg.py:38-47) of x @ W.
__global__ void feature_map_kernel(const double* __restrict__ x, int64_t n, int d,
                                   const double* __restrict__ w1, const double* __restrict__ w2,
                                   int h, double* __restrict__ out) {
  extern __shared__ double sh[];  // [2h] logits + [64] reduction scratch
  double* red = sh + 2 * h;
  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const double* xr = x + row * d;
    for (int f = threadIdx.x; f < 2 * h; f += blockDim.x) {
      const double* w = f < h ? w1 : w2;
      int col = f < h ? f : f - h;
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc = fma(xr[c], w[(int64_t)c * h + col], acc);
      sh[f] = acc;
    }
    __syncthreads();
    for (int half = 0; half < 2; ++half) {
      double* s = sh + half * h;
      double m = -INFINITY;
      for (int f = threadIdx.x; f < h; f += blockDim.x) m = fmax(m, s[f]);
      m = warp_max_d(m);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x == 0) {
        double mm = red[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mm = fmax(mm, red[w]);
        red[32] = mm;
      }
      __syncthreads();
      m = red[32];
      double sum = 0.0;
      for (int f = threadIdx.x; f < h; f += blockDim.x) {
        double e = exp(s[f] - m);
        s[f] = e;
        sum += e;
      }
      sum = warp_sum_d(sum);
      __syncthreads();
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
      __syncthreads();
      if (threadIdx.x == 0) {
        double ss = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ss += red[w];
        red[33] = ss;
      }
      __syncthreads();
      double tot = red[33];
      for (int f = threadIdx.x; f < h; f += blockDim.x) out[row * 2 * h + half * h + f] = s[f] / tot;
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------- state update --
// cache.py:155-158: for i in append order, S += outer(v_q[i], phi[i]),
// P += phi[i].  Each S element is a sequential fp64 sum of separately rounded
// products — the same operation sequence numpy performs.
__global__ void state_update_kernel(const double* __restrict__ vq, const double* __restrict__ phi,
                                    int n, int d, int rank, double* __restrict__ S,
                                    double* __restrict__ P) {
  int64_t total = (int64_t)d * rank + rank;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < (int64_t)d * rank) {
      int c = (int)(i / rank), f = (int)(i % rank);
      double acc = S[i];
      for (int t = 0; t < n; ++t)
        acc = __dadd_rn(acc, __dmul_rn(vq[(int64_t)t * d + c], phi[(int64_t)t * rank + f]));
      S[i] = acc;
    } else {
      int f = (int)(i - (int64_t)d * rank);
      double acc = P[f];
      for (int t = 0; t < n; ++t) acc = __dadd_rn(acc, phi[(int64_t)t * rank + f]);
      P[f] = acc;
    }
  }
}

// ------------------------------------------------------- causal attention --
// One block per query row t over keys i <= t, float64 (attention.py:50-57, 99-155):
//   shifted = 1: attention_reference, softmax of the masked logits (max-shifted,
//     linalg.py:38-47); `weights` (optional) receives the [n][n] softmax rows.
//   shifted = 0: the corrected forms, raw exponentials plus f = phi_q(q_t) . phi_k(k_err_i)
//     (phq / phk [n][rank], NULL without adapter): out = sum (e + f) v / sum (e + f).
// Keys are processed in tiles of blockDim: the weights of a tile go to shared memory,
// then thread c accumulates channel c of the numerator.
__global__ void attn_rows_kernel(const double* __restrict__ q, const double* __restrict__ k,
                                 const double* __restrict__ v, int64_t n, int d,
                                 const double* __restrict__ phq, const double* __restrict__ phk, int rank,
                                 int shifted, double* __restrict__ weights, double* __restrict__ out) {
  extern __shared__ double ash[];  // [blockDim] tile weights, [64] reduction scratch, [d] numerator
  double* wt = ash;
  double* red = ash + blockDim.x;
  double* num = red + 64;
  const int64_t t = blockIdx.x;
  const int tid = threadIdx.x, nwarp = blockDim.x >> 5;
  const double inv = 1.0 / sqrt((double)d);
  const double* qt = q + t * d;
  auto logit = [&](int64_t i) {
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc = fma(qt[c], k[i * d + c], acc);
    return acc * inv;
  };
  double m = 0.0;
  if (shifted) {
    double mx = -INFINITY;
    for (int64_t i = tid; i <= t; i += blockDim.x) mx = fmax(mx, logit(i));
    mx = warp_max_d(mx);
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    m = red[0];
    for (int w = 1; w < nwarp; ++w) m = fmax(m, red[w]);
    __syncthreads();
  }
  for (int c = tid; c < d; c += blockDim.x) num[c] = 0.0;
  double den = 0.0;  // per-thread partial (its keys)
  for (int64_t i0 = 0; i0 <= t; i0 += blockDim.x) {
    const int64_t i = i0 + tid;
    double w = 0.0;
    if (i <= t) {
      w = exp(logit(i) - m);
      if (phq) {
        double f = 0.0;
        for (int r = 0; r < rank; ++r) f = fma(phq[t * rank + r], phk[i * rank + r], f);
        w += f;
      }
    }
    den += w;
    wt[tid] = w;
    __syncthreads();
    const int cnt = (int)(t + 1 - i0 < (int64_t)blockDim.x ? t + 1 - i0 : (int64_t)blockDim.x);
    for (int c = tid; c < d; c += blockDim.x) {
      double acc = num[c];
      for (int j = 0; j < cnt; ++j) acc = fma(wt[j], v[(i0 + j) * d + c], acc);
      num[c] = acc;
    }
    if (weights && i <= t) weights[t * n + i] = w;  // normalised below
    __syncthreads();
  }
  den = warp_sum_d(den);
  if ((tid & 31) == 0) red[tid >> 5] = den;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < nwarp; ++w) tot += red[w];
  for (int c = tid; c < d; c += blockDim.x) out[t * d + c] = num[c] / tot;
  if (weights)
    for (int64_t i = tid; i < n; i += blockDim.x) weights[t * n + i] = i <= t ? weights[t * n + i] / tot : 0.0;
}

__global__ void cast_f64_f32_kernel(const double* __restrict__ q, int d, float* __restrict__ o) {
  for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = (float)q[i];
}

__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dsub_rn(a[i], b[i]);
}

// ------------------------------------------------------------------ decode --
struct RefCache {
  int d, group, bits, lb, lanes, kw, vw, vg;
  uint32_t mask;
  int64_t nq, nr;
  const uint32_t *kwords, *vwords;
  const double *kscales, *kzeros, *vscales, *vzeros, *rk, *rv;
};

// Dequantized key element (cache.py:97-105 -> quantize.py:174-180) as the
// reference computes it (fp64), then cast to float32 (attention.py:242).
__device__ __forceinline__ float key_elem(const RefCache& c, int64_t t, int ch) {
  int64_t ci = t / c.group, ri = t % c.group;
  const uint32_t* w = c.kwords + ci * (int64_t)c.kw * c.d;
  uint32_t code = (w[(ri / c.lanes) * c.d + ch] >> (c.lb * (ri % c.lanes))) & c.mask;
  return (float)__dadd_rn(__dmul_rn((double)code, c.kscales[ci * c.d + ch]), c.kzeros[ci * c.d + ch]);
}

__device__ __forceinline__ float value_elem(const RefCache& c, int64_t t, int ch) {
  uint32_t code = (c.vwords[t * c.vw + ch / c.lanes] >> (c.lb * (ch % c.lanes))) & c.mask;
  int64_t mi = t * c.vg + ch / c.group;
  return (float)__dadd_rn(__dmul_rn((double)code, c.vscales[mi]), c.vzeros[mi]);
}

// logits s_t = (k_t . q32) * inv_sqrt_d in float32 (attention.py:243, 253).
__global__ void ref_logits_kernel(RefCache c, const float* __restrict__ q32, float inv_sqrt_d,
                                  float* __restrict__ logits) {
  int64_t total = c.nq + c.nr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    if (t < c.nq) {
      for (int ch = 0; ch < c.d; ++ch) acc = __fadd_rn(acc, __fmul_rn(key_elem(c, t, ch), q32[ch]));
    } else {
      const double* k = c.rk + (t - c.nq) * c.d;
      for (int ch = 0; ch < c.d; ++ch) acc = __fadd_rn(acc, __fmul_rn((float)k[ch], q32[ch]));
    }
    logits[t] = __fmul_rn(acc, inv_sqrt_d);
  }
}

// One block per decode block (attention.py:238-258): m = max, e = exp(s-m),
// y = e @ v (fp32), l = sum(e).  Block nb (last) is the residual window.
__global__ void ref_block_kernel(RefCache c, int block, int nbq, const float* __restrict__ logits,
                                 float* __restrict__ ys, float* __restrict__ ms, float* __restrict__ ls) {
  int b = blockIdx.x;
  int64_t lo, hi;
  bool raw = b >= nbq;
  if (!raw) {
    lo = (int64_t)b * block;
    hi = min(c.nq, lo + block);
  } else {
    lo = c.nq;
    hi = c.nq + c.nr;
  }
  __shared__ float sm_m, sm_l;
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    for (int64_t t = lo; t < hi; ++t) m = fmaxf(m, logits[t]);
    float l = 0.f;
    for (int64_t t = lo; t < hi; ++t) l = __fadd_rn(l, expf(logits[t] - m));
    sm_m = m;
    sm_l = l;
  }
  __syncthreads();
  float m = sm_m;
  for (int ch = threadIdx.x; ch < c.d; ch += blockDim.x) {
    float acc = 0.f;
    for (int64_t t = lo; t < hi; ++t) {
      float e = expf(logits[t] - m);
      float v = raw ? (float)c.rv[(t - c.nq) * c.d + ch] : value_elem(c, t, ch);
      acc = __fadd_rn(acc, __fmul_rn(e, v));
    }
    ys[(int64_t)b * c.d + ch] = acc;
  }
  if (threadIdx.x == 0) {
    ms[b] = m;
    ls[b] = sm_l;
  }
}

// corr_num = float32(S @ phi), corr_den = float32(P . phi)  (attention.py:224-228)
__global__ void ref_corr_kernel(const double* __restrict__ S, const double* __restrict__ P,
                                const double* __restrict__ phi, int d, int rank,
                                float* __restrict__ cnum, float* __restrict__ cden) {
  for (int c = threadIdx.x; c <= d; c += blockDim.x) {
    const double* row = c < d ? S + (int64_t)c * rank : P;
    double acc = 0.0;
    for (int f = 0; f < rank; ++f) acc = fma(row[f], phi[f], acc);
    if (c < d) cnum[c] = (float)acc;
    else *cden = (float)acc;
  }
}

// _reduce_blocks (attention.py:158-194) + un-rotation + divide (:262-267).
// Single block; thread ch owns channel ch.  Blocks reduce in ascending order.
__global__ void ref_reduce_kernel(int d, int nbq, int has_raw, const float* __restrict__ ys,
                                  const float* __restrict__ ms, const float* __restrict__ ls,
                                  const float* __restrict__ cnum, const float* __restrict__ cden_p,
                                  int use_corr, int literal, int rotated, float* __restrict__ tmp,
                                  double* __restrict__ out) {
  __shared__ float sh_big, sh_den, sh_s;
  __shared__ int sh_mode;
  int nb = nbq + has_raw;
  if (threadIdx.x == 0) {
    float big = -INFINITY;
    for (int j = 0; j < nb; ++j) big = fmaxf(big, ms[j]);
    float dq = 0.f, dr = 0.f;
    for (int j = 0; j < nbq; ++j) dq = __fadd_rn(dq, __fmul_rn(expf(ms[j] - big), ls[j]));
    if (has_raw) dr = __fmul_rn(expf(ms[nbq] - big), ls[nbq]);
    float den = __fadd_rn(dq, dr);
    int mode = 0;  // 0: no correction; 1: literal; 2: M>=0 scale corr; 3: M<0 scale blocks
    float s = 1.f;
    float cden = use_corr ? *cden_p : 0.f;
    bool any = false;
    if (use_corr) {
      any = cden != 0.f;
      for (int ch = 0; ch < d && !any; ++ch) any = cnum[ch] != 0.f;
    }
    if (any) {
      if (literal) {
        mode = 1;
        den = __fadd_rn(den, cden);
      } else if (big >= 0.f) {
        mode = 2;
        s = expf(-big);
        den = __fadd_rn(den, __fmul_rn(s, cden));
      } else {
        mode = 3;
        s = expf(big);
        den = __fadd_rn(__fmul_rn(s, den), cden);
      }
    }
    sh_big = big;
    sh_den = den;
    sh_s = s;
    sh_mode = mode;
  }
  __syncthreads();
  float big = sh_big, s = sh_s;
  int mode = sh_mode;
  for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
    float nq = 0.f, nr = 0.f;
    for (int j = 0; j < nbq; ++j) nq = __fadd_rn(nq, __fmul_rn(expf(ms[j] - big), ys[(int64_t)j * d + ch]));
    if (has_raw) nr = __fmul_rn(expf(ms[nbq] - big), ys[(int64_t)nbq * d + ch]);
    if (mode == 1) nq = __fadd_rn(nq, cnum[ch]);
    else if (mode == 2) nq = __fadd_rn(nq, __fmul_rn(s, cnum[ch]));
    else if (mode == 3) {
      nq = __fadd_rn(__fmul_rn(s, nq), cnum[ch]);
      nr = __fmul_rn(s, nr);
    }
    tmp[ch] = nq;
    tmp[d + ch] = nr;
  }
  __syncthreads();
  // num = num_q @ H32^T + num_r  (H symmetric; entries fp32(+-1/sqrt(d)))
  float h = (float)(1.0 / sqrt((double)d));
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    float num;
    if (rotated) {
      num = 0.f;
      for (int j = 0; j < d; ++j) {
        float sgn = (__popc((unsigned)(j & k)) & 1) ? -h : h;
        num = __fadd_rn(num, __fmul_rn(tmp[j], sgn));
      }
      num = __fadd_rn(num, tmp[d + k]);
    } else {
      num = __fadd_rn(tmp[k], tmp[d + k]);
    }
    out[k] = (double)__fdiv_rn(num, sh_den);
  }
}

}  // namespace
}  // namespace kvlc

using namespace kvlc;

extern "C" {

int kvlc_ref_pack(const uint8_t* codes, int64_t rows, int64_t n, int bits, uint32_t* words,
                  void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(valid_bits(bits), "cannot pack %d-bit codes, supported: [2, 3, 4, 8]", bits);
  int64_t nw = cdiv(n, lanes_per_word(bits));
  if (rows * nw == 0) return KVLC_OK;
  pack_rows_kernel<<<blocks_for(rows * nw), kThreads, 0, as_stream(stream)>>>(
      codes, rows, n, lane_bits(bits), lanes_per_word(bits), words);
  return check_launch("pack");
}

int kvlc_ref_unpack(const uint32_t* words, int64_t rows, int64_t nwords, int64_t count, int bits,
                    uint8_t* codes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(valid_bits(bits), "cannot unpack %d-bit codes, supported: [2, 3, 4, 8]", bits);
  KVLC_REQUIRE(count <= nwords * lanes_per_word(bits), "count %lld exceeds capacity of %lld words",
               (long long)count, (long long)nwords);
  if (rows * count == 0) return KVLC_OK;
  unpack_kernel<<<blocks_for(rows * count), kThreads, 0, as_stream(stream)>>>(
      words, rows, nwords, count, lane_bits(bits), lanes_per_word(bits), (1u << bits) - 1u, codes);
  return check_launch("unpack");
}

int kvlc_ref_quantize(const double* x, int64_t rows, int64_t cols, int bits, int group, int axis,
                      uint32_t* words, double* scales, double* zeros, uint8_t* codes_scratch,
                      void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(valid_bits(bits), "bits must be one of (2, 3, 4, 8), got %d", bits);
  KVLC_REQUIRE(group >= 1, "group_size must be >= 1, got %d", group);
  KVLC_REQUIRE(rows > 0 && cols > 0, "expected a non-empty matrix, got shape (%lld, %lld)",
               (long long)rows, (long long)cols);
  KVLC_REQUIRE(axis == KVLC_AXIS_TOKEN || axis == KVLC_AXIS_CHANNEL, "axis must be token or channel");
  cudaStream_t s = as_stream(stream);
  int top = (1 << bits) - 1;
  int64_t lines = axis == KVLC_AXIS_TOKEN ? rows : cols;
  int64_t ngroups = cdiv(axis == KVLC_AXIS_TOKEN ? cols : rows, group);
  quantize_groups_kernel<<<blocks_for(lines * ngroups), kThreads, 0, s>>>(
      x, rows, cols, group, top, axis, scales, zeros, codes_scratch);
  int lb = lane_bits(bits), lanes = lanes_per_word(bits);
  if (axis == KVLC_AXIS_TOKEN) {
    pack_rows_kernel<<<blocks_for(rows * cdiv(cols, lanes)), kThreads, 0, s>>>(
        codes_scratch, rows, cols, lb, lanes, words);
  } else {
    pack_cols_kernel<<<blocks_for(cdiv(rows, lanes) * cols), kThreads, 0, s>>>(
        codes_scratch, rows, cols, lb, lanes, words);
  }
  return check_launch("quantize");
}

int kvlc_ref_dequantize(const uint32_t* words, const double* scales, const double* zeros,
                        int64_t rows, int64_t cols, int bits, int group, int axis, double* out,
                        void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(valid_bits(bits), "bits must be one of (2, 3, 4, 8), got %d", bits);
  if (rows * cols == 0) return KVLC_OK;
  dequantize_kernel<<<blocks_for(rows * cols), kThreads, 0, as_stream(stream)>>>(
      words, scales, zeros, rows, cols, group, lane_bits(bits), lanes_per_word(bits),
      (1u << bits) - 1u, axis, out);
  return check_launch("dequantize");
}

int kvlc_ref_rotate(const double* x, int64_t rows, int64_t cols, int placement, double* out,
                    void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(placement == KVLC_PLACE_PRE || placement == KVLC_PLACE_POST,
               "placement must be 'pre' or 'post'");
  int64_t dim = placement == KVLC_PLACE_POST ? cols : rows;
  KVLC_REQUIRE(pow2(dim) && dim <= 4096, "Hadamard dimension must be a power of two, got %lld",
               (long long)dim);
  int64_t lines = placement == KVLC_PLACE_POST ? rows : cols;
  if (lines == 0) return KVLC_OK;
  int64_t sl = placement == KVLC_PLACE_POST ? cols : 1;
  int64_t se = placement == KVLC_PLACE_POST ? 1 : cols;
  rotate_dense_kernel<<<blocks_for(lines * dim), kThreads, 0, as_stream(stream)>>>(x, lines, (int)dim, sl, se, out);
  return check_launch("rotate");
}

int kvlc_ref_feature_map(const double* x, int64_t n, int d, const double* w1, const double* w2,
                         int h, double* out, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(d >= 1 && h >= 1, "feature input dim %d / rank half %d invalid", d, h);
  if (n == 0) return KVLC_OK;
  int grid = (int)(n < 65535 ? n : 65535);
  size_t smem = (2 * (size_t)h + 64) * sizeof(double);
  KVLC_REQUIRE(smem <= 48 * 1024, "rank %d too large for the feature-map kernel", 2 * h);
  feature_map_kernel<<<grid, 256, smem, as_stream(stream)>>>(x, n, d, w1, w2, h, out);
  return check_launch("feature_map");
}

int kvlc_ref_attention(const double* q, const double* k, const double* v, int64_t n, int d, const double* phq,
                       const double* phk, int rank, int shifted, double* weights, double* out, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(n >= 0 && d >= 1, "Q/K/V shapes (%lld, %d) invalid", (long long)n, d);
  KVLC_REQUIRE(!phq == !phk && (!phq || rank >= 1), "feature matrices must come together");
  if (n == 0) return KVLC_OK;
  const int threads = 128;
  const size_t smem = ((size_t)threads + 64 + d) * sizeof(double);
  KVLC_REQUIRE(smem <= 48 * 1024, "head dim %d too large for the attention kernel", d);
  KVLC_REQUIRE(n <= 2147483647, "sequence too long");
  attn_rows_kernel<<<(unsigned)n, threads, smem, as_stream(stream)>>>(q, k, v, n, d, phq, phk, rank, shifted ? 1 : 0,
                                                                     weights, out);
  return check_launch("attention");
}

size_t kvlc_ref_flush_scratch(int d, int group, int rank) {
  size_t gd = (size_t)group * d;
  return align_up(gd) + 6 * align_up(gd * sizeof(double)) + align_up((size_t)group * rank * sizeof(double));
}

int kvlc_ref_flush(const double* k_blk, const double* v_blk, int d, int group, int bits, int rotate,
                   const double* w1k, const double* w2k, int rank, uint32_t* kwords,
                   double* kscales, double* kzeros, uint32_t* vwords, double* vscales,
                   double* vzeros, double* s_state, double* p_state, void* scratch, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(d >= 1 && group >= 1, "bad flush shape d=%d group=%d", d, group);
  KVLC_REQUIRE(!rotate || pow2(d), "Hadamard dimension must be a power of two, got %d", d);
  cudaStream_t s = as_stream(stream);
  Arena ar(scratch, kvlc_ref_flush_scratch(d, group, w1k ? rank : 0));
  size_t gd = (size_t)group * d;
  uint8_t* codes = ar.take<uint8_t>(gd);
  double* khat = ar.take<double>(gd);
  double* kerr = ar.take<double>(gd);
  double* vrot = ar.take<double>(gd);
  double* vq = ar.take<double>(gd);
  double* spare1 = ar.take<double>(gd);
  double* spare2 = ar.take<double>(gd);
  (void)spare1;
  (void)spare2;
  KVLC_REQUIRE(codes && khat && kerr && vrot && vq, "flush scratch too small");
  int rc;
  // keys: channel-wise, one group per channel (cache.py:141)
  if ((rc = kvlc_ref_quantize(k_blk, group, d, bits, group, KVLC_AXIS_CHANNEL, kwords, kscales,
                              kzeros, codes, stream)))
    return rc;
  // values: Hadamard post-rotation then token-wise (cache.py:143-145)
  const double* vstore = v_blk;
  if (rotate) {
    if ((rc = kvlc_ref_rotate(v_blk, group, d, KVLC_PLACE_POST, vrot, stream))) return rc;
    vstore = vrot;
  }
  if ((rc = kvlc_ref_quantize(vstore, group, d, bits, group, KVLC_AXIS_TOKEN, vwords, vscales,
                              vzeros, codes, stream)))
    return rc;
  if (w1k == nullptr) return KVLC_OK;
  KVLC_REQUIRE(rank >= 2 && rank % 2 == 0, "rank must be an even integer >= 2, got %d", rank);
  double* phi = ar.take<double>((size_t)group * rank);
  KVLC_REQUIRE(phi, "flush scratch too small");
  // k_err = k - K_hat, v_q = dequantized stored values (cache.py:153-154)
  if ((rc = kvlc_ref_dequantize(kwords, kscales, kzeros, group, d, bits, group, KVLC_AXIS_CHANNEL,
                                khat, stream)))
    return rc;
  sub_kernel<<<blocks_for(gd), kThreads, 0, s>>>(k_blk, khat, (int64_t)gd, kerr);
  if ((rc = kvlc_ref_dequantize(vwords, vscales, vzeros, group, d, bits, group, KVLC_AXIS_TOKEN, vq,
                                stream)))
    return rc;
  if ((rc = kvlc_ref_feature_map(kerr, group, d, w1k, w2k, rank / 2, phi, stream))) return rc;
  state_update_kernel<<<blocks_for((int64_t)d * rank + rank), kThreads, 0, s>>>(vq, phi, group, d, rank,
                                                                              s_state, p_state);
  return check_launch("flush state update");
}

size_t kvlc_ref_decode_scratch(int d, int64_t nq, int64_t nr, int block, int rank) {
  int64_t nb = (block > 0 ? cdiv(nq, block) : 0) + 1;
  return align_up((nq + nr + 1) * sizeof(float)) + align_up(nb * (size_t)d * sizeof(float)) +
         2 * align_up(nb * sizeof(float)) + align_up((size_t)d * sizeof(float) * 3) +
         align_up(sizeof(float) * 4) + align_up((size_t)(rank + 2) * sizeof(double)) +
         align_up((size_t)d * sizeof(float));
}

int kvlc_ref_decode(const double* q, int d, int group, int bits, int rotated, int64_t n_chunks,
                    const uint32_t* kwords, const double* kscales, const double* kzeros,
                    const uint32_t* vwords, const double* vscales, const double* vzeros,
                    int64_t nr, const double* rk, const double* rv, const double* w1q,
                    const double* w2q, const double* s_state, const double* p_state, int rank,
                    int block_tokens, int literal, double* out, float* part_y, float* part_m,
                    float* part_l, void* scratch, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(block_tokens >= 1, "block_tokens must be >= 1, got %d", block_tokens);
  int64_t nq = n_chunks * group;
  KVLC_REQUIRE(nq + nr > 0, "cannot decode against an empty cache");
  cudaStream_t s = as_stream(stream);
  RefCache c;
  c.d = d;
  c.group = group;
  c.bits = bits;
  c.lb = lane_bits(bits);
  c.lanes = lanes_per_word(bits);
  c.kw = (int)cdiv(group, c.lanes);
  c.vw = (int)cdiv(d, c.lanes);
  c.vg = (int)cdiv(d, group);
  c.mask = (1u << bits) - 1u;
  c.nq = nq;
  c.nr = nr;
  c.kwords = kwords;
  c.vwords = vwords;
  c.kscales = kscales;
  c.kzeros = kzeros;
  c.vscales = vscales;
  c.vzeros = vzeros;
  c.rk = rk;
  c.rv = rv;
  int nbq = (int)cdiv(nq, block_tokens);
  int has_raw = nr > 0 ? 1 : 0;
  int nb = nbq + has_raw;
  bool use_corr = w1q != nullptr && s_state != nullptr;
  Arena ar(scratch, kvlc_ref_decode_scratch(d, nq, nr, block_tokens, use_corr ? rank : 0));
  float* logits = ar.take<float>(nq + nr + 1);
  float* ys = ar.take<float>((size_t)(nbq + 1) * d);
  float* ms = ar.take<float>(nbq + 1);
  float* ls = ar.take<float>(nbq + 1);
  float* cnum = ar.take<float>((size_t)d * 3);
  float* cden = ar.take<float>(4);
  double* phi = ar.take<double>(rank + 2);
  KVLC_REQUIRE(logits && ys && ms && ls && cnum && cden, "decode scratch too small");
  float* tmp = cnum + d;
  int rc;
  if (use_corr) {
    KVLC_REQUIRE(phi != nullptr, "decode scratch too small");
    if ((rc = kvlc_ref_feature_map(q, 1, d, w1q, w2q, rank / 2, phi, stream))) return rc;
    ref_corr_kernel<<<1, 256, 0, s>>>(s_state, p_state, phi, d, rank, cnum, cden);
  }
  float* q32buf = ar.take<float>(d);
  KVLC_REQUIRE(q32buf, "decode scratch too small");
  cast_f64_f32_kernel<<<1, 256, 0, s>>>(q, d, q32buf);
  float inv_sqrt_d = (float)(1.0 / sqrt((double)d));
  ref_logits_kernel<<<blocks_for(nq + nr, 128), 128, 0, s>>>(c, q32buf, inv_sqrt_d, logits);
  ref_block_kernel<<<nb, 128, 0, s>>>(c, block_tokens, nbq, logits, ys, ms, ls);
  ref_reduce_kernel<<<1, 256, 0, s>>>(d, nbq, has_raw, ys, ms, ls, cnum, cden, use_corr ? 1 : 0,
                                      literal, rotated, tmp, out);
  if (part_y) KVLC_CUDA(cudaMemcpyAsync(part_y, ys, (size_t)nb * d * sizeof(float), cudaMemcpyDeviceToDevice, s));
  if (part_m) KVLC_CUDA(cudaMemcpyAsync(part_m, ms, (size_t)nb * sizeof(float), cudaMemcpyDeviceToDevice, s));
  if (part_l) KVLC_CUDA(cudaMemcpyAsync(part_l, ls, (size_t)nb * sizeof(float), cudaMemcpyDeviceToDevice, s));
  return check_launch("decode");
}

}  // extern "C"
