// Serving-path cache writers: prefill, per-step append and the fused flush
// (K1 channel-wise key quantization, K2 FWHT + token-wise value quantization,
// K3 adapter-state update) for the batched [B, Hkv] cache, d = G = 128.
//
// Reference: KVCacheState.append / flush_group (cache.py:120-158),
// quantize_tensor (quantize.py:189-239), rotate (hadamard.py:45-57),
// phi_k / feature_map (adapter.py:80-96).
//
// Code decisions are bit-exact with the reference: float64 min / max, scale
// (max-min)/3 and (x-min)/scale rounded half-to-even.  The division is done
// as a float64 reciprocal multiply and re-done as an IEEE division only when
// the quotient lies within 1e-9 of a rounding boundary, which gives the
// division's result whenever it matters.  Metadata is stored as
// float16(fp64 value).  k_err / v_q for the state update use the float64
// scales, as cache.py:153-154 does.
#include <type_traits>

#include "kvlc_common.cuh"
#include "kvlc_tc.cuh"

#include <algorithm>
#include <cstring>

namespace kvlc {
namespace {

constexpr int D = KVLC_D;
constexpr int G = KVLC_G;
constexpr int SLOTS = KVLC_SLOTS;
constexpr int RANK = KVLC_RANK;
constexpr int HALF = RANK / 2;
constexpr int KERR_LD = D + 1;  // padded row (bank-conflict free column reads)
constexpr int FLUSH_THREADS = 256;
constexpr size_t FLUSH_SMEM = (size_t)G * KERR_LD * 4 + (size_t)G * D * 4 + (size_t)G * HALF * 4;

__device__ __forceinline__ float bf2f(uint16_t x) { return __uint_as_float((uint32_t)x << 16); }

// code = rint((x - mn) / scale) with the reference's IEEE-division result.
__device__ __forceinline__ uint32_t code2(double x, double mn, double scale, double inv) {
  if (!(scale > 0.0)) return 0u;
  double diff = __dsub_rn(x, mn);
  double r = diff * inv;
  double fr = r - floor(r);
  if (fabs(fr - 0.5) < 1e-9) r = __ddiv_rn(diff, scale);  // near a tie: exact division
  r = rint(r);
  r = fmin(fmax(r, 0.0), 3.0);
  return (uint32_t)r;
}

// True when float16 rounding of x could differ between two evaluations of x
// that agree to ~1e-12 relative (x sits next to an fp16 rounding midpoint).
__device__ __forceinline__ bool near_half_tie(double x) {
  return __half_as_ushort(__double2half(x * (1.0 - 1e-12))) !=
         __half_as_ushort(__double2half(x * (1.0 + 1e-12)));
}

// ---- fragment-native code layouts (include/kvlinc.h, consumed by kvlc_decode.cu) ----
// Key word wi = ((w*32 + lane)*8 + kt), lane = 4g + t0: byte q holds channel
// 16kt + 2t0 + {0,8,1,9}[q]; its bit pair j holds token 32w + 4g + j.
__device__ __forceinline__ uint32_t pack_k_word(const uint8_t* codes, int wi) {
  const int kt = wi & 7, lane = (wi >> 3) & 31, w = wi >> 8;
  const int g = lane >> 2, t0 = lane & 3;
  const int coff[4] = {0, 8, 1, 9};
  uint32_t word = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      word |= (uint32_t)codes[(32 * w + 4 * g + j) * D + 16 * kt + 2 * t0 + coff[q]] << (8 * q + 2 * j);
  return word;
}

// Value word wi = ((w*32 + lane)*8 + 4mt + p), lane = 4g + t0: byte q holds
// token 32w + 8t0 + 2mt + {0,1,4,5}[q]; its bit pair j holds channel 32p + 8j + g.
__device__ __forceinline__ uint32_t pack_v_word(const uint8_t* codes, int wi) {
  const int i = wi & 7, lane = (wi >> 3) & 31, w = wi >> 8;
  const int g = lane >> 2, t0 = lane & 3, mt = i >> 2, p = i & 3;
  const int toff[4] = {0, 1, 4, 5};
  uint32_t word = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      word |= (uint32_t)codes[(32 * w + 8 * t0 + 2 * mt + toff[q]) * D + 32 * p + 8 * j + g] << (8 * q + 2 * j);
  return word;
}

// Code of (token t, channel c) of one chunk, from the device layouts above.
__device__ __forceinline__ uint32_t k_code(const uint32_t* words, int t, int c) {
  const int w = t >> 5, u = t & 31, g = u >> 2, j = u & 3;
  const int kt = c >> 4, cc = c & 15, t0 = (cc & 7) >> 1, q = ((cc & 1) << 1) | (cc >> 3);
  return (frag_load(words[((w * 32) + 4 * g + t0) * 8 + kt]) >> (8 * q + 2 * j)) & 3u;
}

__device__ __forceinline__ uint32_t v_code(const uint32_t* words, int t, int c) {
  const int w = t >> 5, u = t & 31, t0 = u >> 3, hi = (u >> 2) & 1, mt = (u >> 1) & 1, lo = u & 1;
  const int q = lo + 2 * hi, g = c & 7, r = (c >> 3) & 1, mv = c >> 4, p = mv >> 1, j = 2 * (mv & 1) + r;
  return (frag_load(words[((w * 32) + 4 * g + t0) * 8 + 4 * mt + p]) >> (8 * q + 2 * j)) & 3u;
}

constexpr int MAX_B = 1024;

// Per-sequence host data passed by value (no H2D copy, graph-capturable).
struct SeqInfo {
  int32_t nflush[MAX_B];  // prefill: chunks to flush per sequence
  int32_t len[MAX_B];     // prefill: tokens per sequence
  uint32_t active[MAX_B / 32];  // append: sequence appends this step
  uint32_t flush[MAX_B / 32];   // append: sequence flushes after appending
  __device__ __forceinline__ bool is_active(int b) const { return (active[b >> 5] >> (b & 31)) & 1u; }
  __device__ __forceinline__ bool is_flush(int b) const { return (flush[b >> 5] >> (b & 31)) & 1u; }
};

struct FlushArgs {
  kvlc_cache c;
  kvlc_adapter ad;
  int use_adapter;
  // token source: element (t, ch) of unit u's chunk at
  //   src + u*src_unit + chunk_tok0*src_t + t*src_t + ch*src_c
  const uint16_t* ksrc;
  const uint16_t* vsrc;
  int64_t k_unit, k_t, k_c;
  int64_t v_unit, v_t, v_c;
  int ring;                  // 1: source = residual ring, token t at slot res_start + t
  int cpc;                   // chunks per CTA (prefill)
  float* s_out;              // prefill: per-CTA S partial [units][splits][D][RANK]; null => cache S
  float* p_out;
  int splits;
  // prefill tensor-core path: quant_kernel -> state kernel operand images (the state
  // kernel's shared-memory tiles byte for byte), slot = unit * slot_stride + chunk
  uint8_t* aimg;             // [slot][hi, lo][FT_TILE]  k_err = A_phi (MN-major, 128 B swizzle)
  uint8_t* cimg;             // [slot][FT_TILE]  value codes as fp16, [M = channel][K = token] MN-major
  float2* vsz;               // [slot][G]  value (scale, zero) per token, fp32 (v_q = s code + z)
  int slot_stride;
  // quant_kernel work split (decode-time ring flushes: one chunk per unit, latency-bound):
  // 0 = one CTA per chunk does K1 and K2; n > 0 = blockIdx.z 0 does K1, z = 1..n do K2 on
  // the tokens of 32-token slice z - 1 (n = G / 32)
  int vsplit;
  // the phi GEMM W tiles, prepared by quant_kernel's first CTAs (no separate launch)
  uint8_t* wtiles;
  int prep_n;                // 16 * Hkv * 2 blocks of 256 threads, 0 = none
  int finalize;              // flush_tc_kernel CTA 0 applies append_finalize (ring flushes)
  int both;                  // flush_tc_kernel: one CTA per unit runs both feature halves (one chunk)
};

__global__ void __launch_bounds__(FLUSH_THREADS, 1) flush_kernel(const FlushArgs a, const SeqInfo seq) {
  extern __shared__ __align__(16) float smem[];
  float* kerr = smem;                       // [G][KERR_LD]
  float* vq = kerr + G * KERR_LD;           // [G][D]  (rotated basis)
  float* phi = vq + G * D;                  // [G][HALF]
  uint8_t* codes_s = reinterpret_cast<uint8_t*>(phi);  // [G][D] codes, before phi is live
  const kvlc_cache& c = a.c;
  const int unit = blockIdx.y, split = blockIdx.x;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  int c_lo, c_hi, dst0;
  if (a.ring) {
    if (!seq.is_flush(b)) return;
    c_lo = 0;
    c_hi = 1;
    dst0 = c.n_chunks[b];
  } else {
    int nf = seq.nflush[b];
    c_lo = split * a.cpc;
    c_hi = min(nf, c_lo + a.cpc);
    dst0 = 0;
  }
  if (c_lo >= c_hi) return;

  float* S = a.s_out ? a.s_out + ((size_t)unit * a.splits + split) * D * RANK : c.S + (size_t)unit * D * RANK;
  float* P = a.p_out ? a.p_out + ((size_t)unit * a.splits + split) * RANK : c.P + (size_t)unit * RANK;

  for (int ci = c_lo; ci < c_hi; ++ci) {
    const int dst = dst0 + ci;  // destination chunk index
    int64_t tok0 = a.ring ? c.res_start[b] : (int64_t)ci * G;
    const uint16_t* K = a.ksrc + unit * a.k_unit + tok0 * a.k_t;
    const uint16_t* V = a.vsrc + unit * a.v_unit + tok0 * a.v_t;
    const size_t cb = (size_t)unit * c.max_chunks + dst;

    // ---- K1: keys, channel-wise (one group of G tokens per channel) ----
    {
      const int ch = tid & (D - 1), half = tid >> 7;  // 2 threads per channel
      float mnf = INFINITY, mxf = -INFINITY;
      for (int t = half * 64; t < half * 64 + 64; ++t) {
        float x = bf2f(K[t * a.k_t + ch * a.k_c]);
        mnf = fminf(mnf, x);
        mxf = fmaxf(mxf, x);
      }
      __shared__ float red_mn[FLUSH_THREADS], red_mx[FLUSH_THREADS];
      red_mn[tid] = mnf;
      red_mx[tid] = mxf;
      __syncthreads();
      double mn = (double)fminf(red_mn[ch], red_mn[ch + 128]);
      double mx = (double)fmaxf(red_mx[ch], red_mx[ch + 128]);
      double scale = __ddiv_rn(__dsub_rn(mx, mn), 3.0);
      double inv = scale > 0.0 ? 1.0 / scale : 0.0;
#pragma unroll 4
      for (int t = half * 64; t < half * 64 + 64; ++t) {
        const double x = (double)bf2f(K[t * a.k_t + ch * a.k_c]);
        const uint32_t code = code2(x, mn, scale, inv);
        codes_s[t * D + ch] = (uint8_t)code;
        const double khat = __dadd_rn(__dmul_rn((double)code, scale), mn);
        kerr[t * KERR_LD + ch] = (float)__dsub_rn(x, khat);
      }
      if (half == 0) {
        c.kscale[cb * D + ch] = __half_as_ushort(__double2half(scale));
        c.kzero[cb * D + ch] = __half_as_ushort(__double2half(mn));
      }
    }
    __syncthreads();
    // pack the key codes into the decode kernel's fragment-native word layout
    for (int wi = tid; wi < 1024; wi += FLUSH_THREADS) c.kcodes[cb * 1024 + wi] = frag_store(pack_k_word(codes_s, wi));
    __syncthreads();

    // ---- K2: values, FWHT post-rotation (fp64) then token-wise quantization ----
    for (int t = warp; t < G; t += FLUSH_THREADS / 32) {
      double x[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) x[e] = (double)bf2f(V[t * a.v_t + (lane * 4 + e) * a.v_c]);
      // stages 1, 2 inside the lane
      double u0 = x[0] + x[1], u1 = x[0] - x[1], u2 = x[2] + x[3], u3 = x[2] - x[3];
      x[0] = u0 + u2;
      x[2] = u0 - u2;
      x[1] = u1 + u3;
      x[3] = u1 - u3;
      // stages 4..64 across lanes
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          double o = __shfl_xor_sync(0xffffffffu, x[e], k);
          x[e] = fma(x[e], (lane & k) ? -1.0 : 1.0, o);  // o - x or x + o (exact)
        }
      }
      const double hs = 1.0 / sqrt((double)D);
      double mn = INFINITY, mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        x[e] = x[e] * hs;
        mn = fmin(mn, x[e]);
        mx = fmax(mx, x[e]);
      }
      mn = warp_min_d(mn);
      mx = warp_max_d(mx);
      double scale = __ddiv_rn(__dsub_rn(mx, mn), 3.0);
      double inv = scale > 0.0 ? 1.0 / scale : 0.0;
      // The FWHT and the reference's dense x @ H (sequential FMA over j) agree
      // to an ulp; they can only disagree on a code at a rounding tie or on an
      // fp16 rounding of the metadata.  Such tokens are re-evaluated in the
      // reference's exact arithmetic order.
      bool amb = near_half_tie(scale) || near_half_tie(mn);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double r = __dsub_rn(x[e], mn) * inv;
        amb |= scale > 0.0 && fabs(r - floor(r) - 0.5) < 1e-9;
      }
      if (__any_sync(0xffffffffu, amb)) {
        mn = INFINITY;
        mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int ch = lane * 4 + e;
          double acc = 0.0;
          for (int j = 0; j < D; ++j) {
            const double hj = (__popc((unsigned)(j & ch)) & 1) ? -hs : hs;
            acc = fma((double)bf2f(V[t * a.v_t + j * a.v_c]), hj, acc);
          }
          x[e] = acc;
          mn = fmin(mn, acc);
          mx = fmax(mx, acc);
        }
        mn = warp_min_d(mn);
        mx = warp_max_d(mx);
        scale = __ddiv_rn(__dsub_rn(mx, mn), 3.0);
        inv = scale > 0.0 ? 1.0 / scale : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t code = code2(x[e], mn, scale, inv);
        codes_s[t * D + lane * 4 + e] = (uint8_t)code;
        vq[t * D + lane * 4 + e] = (float)__dadd_rn(__dmul_rn((double)code, scale), mn);
      }
      if (lane == 0) {
        c.vscale[cb * G + t] = __half_as_ushort(__double2half(scale));
        c.vzero[cb * G + t] = __half_as_ushort(__double2half(mn));
      }
    }
    __syncthreads();
    for (int wi = tid; wi < 1024; wi += FLUSH_THREADS) c.vcodes[cb * 1024 + wi] = frag_store(pack_v_word(codes_s, wi));
    __syncthreads();
    if (!a.use_adapter) continue;

    // ---- K3: phi_k(k_err) per token (two softmax halves), S += vq^T phi, P += sum phi ----
    const int tr = tid >> 4, fc = tid & 15;  // 16 x 16 thread tile, 8 x 8 outputs each
    for (int hf = 0; hf < 2; ++hf) {
      const float* W = (hf == 0 ? a.ad.w1k : a.ad.w2k) + (size_t)kvh * D * HALF;
      {
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (int ch = 0; ch < D; ++ch) {
          float av[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) av[i] = kerr[(tr * 8 + i) * KERR_LD + ch];
          const float4* wp = reinterpret_cast<const float4*>(W + ch * HALF + fc * 8);
          float4 w0 = __ldg(wp), w1 = __ldg(wp + 1);
          float bv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) phi[(tr * 8 + i) * HALF + fc * 8 + j] = acc[i][j];
      }
      __syncthreads();
      // softmax over the HALF features of each token (one warp per token)
      for (int t = warp; t < G; t += FLUSH_THREADS / 32) {
        float v[4];
        float m = -INFINITY;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[e] = phi[t * HALF + lane + 32 * e];
          m = fmaxf(m, v[e]);
        }
        m = warp_max(m);
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[e] = expf(v[e] - m);
          s += v[e];
        }
        s = warp_sum(s);
        float inv = 1.f / s;
#pragma unroll
        for (int e = 0; e < 4; ++e) phi[t * HALF + lane + 32 * e] = v[e] * inv;
      }
      __syncthreads();
      // S[ch][hf*HALF + f] += sum_t vq[t][ch] * phi[t][f]
      {
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (int t = 0; t < G; ++t) {
          const float4* vp = reinterpret_cast<const float4*>(vq + t * D + tr * 8);
          const float4* pp = reinterpret_cast<const float4*>(phi + t * HALF + fc * 8);
          float4 v0 = vp[0], v1 = vp[1], p0 = pp[0], p1 = pp[1];
          float av[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
          float bv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4* sp = reinterpret_cast<float4*>(S + (size_t)(tr * 8 + i) * RANK + hf * HALF + fc * 8);
          float4 s0 = sp[0], s1 = sp[1];
          s0.x += acc[i][0]; s0.y += acc[i][1]; s0.z += acc[i][2]; s0.w += acc[i][3];
          s1.x += acc[i][4]; s1.y += acc[i][5]; s1.z += acc[i][6]; s1.w += acc[i][7];
          sp[0] = s0;
          sp[1] = s1;
        }
        if (tid < HALF) {
          float ps = 0.f;
          for (int t = 0; t < G; ++t) ps += phi[t * HALF + tid];
          P[hf * HALF + tid] += ps;
        }
      }
      __syncthreads();
    }
  }
}

// Ordered reduction of prefill S/P partials into the cache (deterministic).
__global__ void reduce_state_kernel(kvlc_cache c, const float* __restrict__ s_part,
                                    const float* __restrict__ p_part, int splits) {
  const int unit = blockIdx.y;
  const size_t n = (size_t)D * RANK + RANK;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float acc;
    if (i < (size_t)D * RANK) {
      acc = c.S[(size_t)unit * D * RANK + i];
      for (int s = 0; s < splits; ++s) acc += s_part[((size_t)unit * splits + s) * D * RANK + i];
      c.S[(size_t)unit * D * RANK + i] = acc;
    } else {
      size_t f = i - (size_t)D * RANK;
      acc = c.P[(size_t)unit * RANK + f];
      for (int s = 0; s < splits; ++s) acc += p_part[((size_t)unit * splits + s) * RANK + f];
      c.P[(size_t)unit * RANK + f] = acc;
    }
  }
}

// Residual-window load after prefill: tokens [nflush*G, len) -> slots 0..
__global__ void load_residual_kernel(kvlc_cache c, const uint16_t* __restrict__ k,
                                     const uint16_t* __restrict__ v, int64_t n_tok, const SeqInfo seq) {
  const int unit = blockIdx.y;
  const int b = unit / c.Hkv;
  const int first = seq.nflush[b] * G, cnt = seq.len[b] - first;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt * D; i += gridDim.x * blockDim.x) {
    int t = i / D, ch = i % D;
    size_t src = ((size_t)unit * n_tok + first + t) * D + ch;
    c.kres[((size_t)unit * SLOTS + t) * D + ch] = k[src];
    c.vres[((size_t)unit * D + ch) * SLOTS + t] = v[src];
  }
}

__global__ void set_lengths_kernel(kvlc_cache c, const SeqInfo seq) {
  for (int b = threadIdx.x; b < c.B; b += blockDim.x) {
    c.n_chunks[b] = seq.nflush[b];
    c.res_start[b] = 0;
    c.res_len[b] = seq.len[b] - seq.nflush[b] * G;
  }
}

// append (cache.py:120-126): token into ring slot (start + len) mod 256
__global__ void append_kernel(kvlc_cache c, const uint16_t* __restrict__ k_t,
                              const uint16_t* __restrict__ v_t, const SeqInfo seq) {
  const int unit = blockIdx.x, b = unit / c.Hkv, ch = threadIdx.x;
  if (!seq.is_active(b)) return;
  const int slot = (c.res_start[b] + c.res_len[b]) & (SLOTS - 1);
  c.kres[((size_t)unit * SLOTS + slot) * D + ch] = k_t[(size_t)unit * D + ch];
  c.vres[((size_t)unit * D + ch) * SLOTS + slot] = v_t[(size_t)unit * D + ch];
}

// ring counters after an append (+ flush of the due sequences): cache.py:120-147
__device__ __forceinline__ void append_finalize(const kvlc_cache& c, const SeqInfo& seq) {
  for (int b = threadIdx.x; b < c.B; b += blockDim.x) {
    int len = c.res_len[b] + (seq.is_active(b) ? 1 : 0);
    if (seq.is_flush(b)) {
      len -= G;
      c.res_start[b] = (c.res_start[b] + G) & (SLOTS - 1);
      c.n_chunks[b] += 1;
    }
    c.res_len[b] = len;
  }
}
__global__ void append_finalize_kernel(kvlc_cache c, const SeqInfo seq) { append_finalize(c, seq); }

__global__ void export_chunk_kernel(kvlc_cache c, int unit, int chunk, uint32_t* kw, uint32_t* vw,
                                    uint16_t* ks, uint16_t* kz, uint16_t* vs, uint16_t* vz) {
  const size_t cb = (size_t)unit * c.max_chunks + chunk;
  const uint32_t* kwords = c.kcodes + cb * 1024;
  const uint32_t* vwords = c.vcodes + cb * 1024;
  for (int i = threadIdx.x; i < 8 * 128; i += blockDim.x) {
    // reference key word (w, ch): tokens 16w..16w+15 of channel ch (quantize.py:15-19)
    const int w = i / 128, ch = i % 128;
    uint32_t word = 0;
    for (int l = 0; l < 16; ++l) word |= k_code(kwords, 16 * w + l, ch) << (2 * l);
    kw[i] = word;
    // reference value_rows word (t, j): channels 16j..16j+15 of token t
    const int t = i / 8, j = i % 8;
    word = 0;
    for (int l = 0; l < 16; ++l) word |= v_code(vwords, t, 16 * j + l) << (2 * l);
    vw[i] = word;
  }
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    ks[i] = c.kscale[cb * D + i];
    kz[i] = c.kzero[cb * D + i];
    vs[i] = c.vscale[cb * G + i];
    vz[i] = c.vzero[cb * G + i];
  }
}

// ---------------------------------------------------------------------------
// .kvlc image of one unit (cache.py:197-230, little-endian): header "KVLC" + u32
// (version 1, d, rank, G, R, bits, values_rotated, quantized_tokens, residual_len);
// key chunk words [8][128] per chunk; value_rows words [n_q][8]; per chunk key
// scales then zeros (f16 [128]); value scales [n_q] then zeros [n_q] (f16);
// residual keys then values (f16 [n_res][128], oldest first); S [128][256] then
// P [256] (f16) when rank > 0.  Offsets for n chunks / n_res residual tokens:
struct ImageLayout {
  size_t kcodes, vcodes, kmeta, vscale, vzero, rk, rv, S, P, end;
  __host__ __device__ ImageLayout(int n, int n_res, int rank) {
    kcodes = 40;
    vcodes = kcodes + (size_t)n * 8 * 128 * 4;
    kmeta = vcodes + (size_t)n * G * 8 * 4;
    vscale = kmeta + (size_t)n * 2 * D * 2;
    vzero = vscale + (size_t)n * G * 2;
    rk = vzero + (size_t)n * G * 2;
    rv = rk + (size_t)n_res * D * 2;
    S = rv + (size_t)n_res * D * 2;
    P = S + (rank ? (size_t)D * rank * 2 : 0);
    end = P + (size_t)rank * 2;
  }
};

// grid: n chunk blocks, then one residual / header block, then state blocks.
__global__ void serialize_unit_kernel(kvlc_cache c, int unit, int n, int res_start, int n_res, int rank,
                                      uint8_t* __restrict__ img) {
  const ImageLayout L(n, n_res, rank);
  const int bx = blockIdx.x, tid = threadIdx.x;
  if (bx < n) {
    const size_t cb = (size_t)unit * c.max_chunks + bx;
    const uint32_t* kwords = c.kcodes + cb * 1024;
    const uint32_t* vwords = c.vcodes + cb * 1024;
    uint32_t* kw = reinterpret_cast<uint32_t*>(img + L.kcodes) + (size_t)bx * 1024;
    uint32_t* vw = reinterpret_cast<uint32_t*>(img + L.vcodes) + (size_t)bx * G * 8;
    for (int i = tid; i < 1024; i += blockDim.x) {
      const int w = i / 128, ch = i % 128, t = i / 8, j = i % 8;
      uint32_t kword = 0, vword = 0;
      for (int l = 0; l < 16; ++l) {
        kword |= k_code(kwords, 16 * w + l, ch) << (2 * l);
        vword |= v_code(vwords, t, 16 * j + l) << (2 * l);
      }
      kw[i] = kword;
      vw[i] = vword;
    }
    uint16_t* km = reinterpret_cast<uint16_t*>(img + L.kmeta) + (size_t)bx * 2 * D;
    uint16_t* vs = reinterpret_cast<uint16_t*>(img + L.vscale) + (size_t)bx * G;
    uint16_t* vz = reinterpret_cast<uint16_t*>(img + L.vzero) + (size_t)bx * G;
    for (int i = tid; i < 128; i += blockDim.x) {
      km[i] = c.kscale[cb * D + i];
      km[D + i] = c.kzero[cb * D + i];
      vs[i] = c.vscale[cb * G + i];
      vz[i] = c.vzero[cb * G + i];
    }
  } else if (bx == n) {
    if (tid == 0) {
      const uint32_t hdr[10] = {0x434C564Bu /* "KVLC" */, 1u, (uint32_t)D, (uint32_t)rank, (uint32_t)G, (uint32_t)KVLC_R,
                                2u, 1u, (uint32_t)(n * G), (uint32_t)n_res};
      for (int i = 0; i < 10; ++i) reinterpret_cast<uint32_t*>(img)[i] = hdr[i];
    }
    uint16_t* rk = reinterpret_cast<uint16_t*>(img + L.rk);
    uint16_t* rv = reinterpret_cast<uint16_t*>(img + L.rv);
    for (int i = tid; i < n_res * D; i += blockDim.x) {
      const int t = i / D, ch = i % D, slot = (res_start + t) & (SLOTS - 1);
      const float kf = __uint_as_float((uint32_t)c.kres[((size_t)unit * SLOTS + slot) * D + ch] << 16);
      const float vf = __uint_as_float((uint32_t)c.vres[((size_t)unit * D + ch) * SLOTS + slot] << 16);
      rk[i] = __half_as_ushort(__float2half_rn(kf));
      rv[i] = __half_as_ushort(__float2half_rn(vf));
    }
  } else if (rank) {
    uint16_t* S = reinterpret_cast<uint16_t*>(img + L.S);
    uint16_t* P = reinterpret_cast<uint16_t*>(img + L.P);
    for (int i = (bx - n - 1) * blockDim.x + tid; i < D * RANK + RANK; i += (gridDim.x - n - 1) * blockDim.x) {
      if (i < D * RANK) S[i] = __half_as_ushort(__float2half_rn(c.S[(size_t)unit * D * RANK + i]));
      else P[i - D * RANK] = __half_as_ushort(__float2half_rn(c.P[(size_t)unit * RANK + i - D * RANK]));
    }
  }
}

// deserialize_cache (cache.py:252-307) into the device layouts: reference words ->
// dense code tile in shared memory -> pack_k_word / pack_v_word; residual loaded at
// ring slot 0 (f16 -> bf16, the serving cache's residual precision); S / P from f16
// (zero when rank = 0); the sequence counters of unit / Hkv.
__global__ void deserialize_unit_kernel(kvlc_cache c, int unit, int n, int n_res, int rank,
                                        const uint8_t* __restrict__ img) {
  const ImageLayout L(n, n_res, rank);
  const int bx = blockIdx.x, tid = threadIdx.x;
  if (bx < n) {
    __shared__ uint8_t codes[G * D];
    const size_t cb = (size_t)unit * c.max_chunks + bx;
    const uint32_t* kw = reinterpret_cast<const uint32_t*>(img + L.kcodes) + (size_t)bx * 1024;
    const uint32_t* vw = reinterpret_cast<const uint32_t*>(img + L.vcodes) + (size_t)bx * G * 8;
    for (int i = tid; i < G * D; i += blockDim.x) {
      const int t = i / D, ch = i % D;
      codes[i] = (uint8_t)((kw[(t >> 4) * 128 + ch] >> (2 * (t & 15))) & 3u);
    }
    __syncthreads();
    for (int wi = tid; wi < 1024; wi += blockDim.x) c.kcodes[cb * 1024 + wi] = frag_store(pack_k_word(codes, wi));
    __syncthreads();
    for (int i = tid; i < G * D; i += blockDim.x) {
      const int t = i / D, ch = i % D;
      codes[i] = (uint8_t)((vw[t * 8 + (ch >> 4)] >> (2 * (ch & 15))) & 3u);
    }
    __syncthreads();
    for (int wi = tid; wi < 1024; wi += blockDim.x) c.vcodes[cb * 1024 + wi] = frag_store(pack_v_word(codes, wi));
    const uint16_t* km = reinterpret_cast<const uint16_t*>(img + L.kmeta) + (size_t)bx * 2 * D;
    const uint16_t* vs = reinterpret_cast<const uint16_t*>(img + L.vscale) + (size_t)bx * G;
    const uint16_t* vz = reinterpret_cast<const uint16_t*>(img + L.vzero) + (size_t)bx * G;
    for (int i = tid; i < 128; i += blockDim.x) {
      c.kscale[cb * D + i] = km[i];
      c.kzero[cb * D + i] = km[D + i];
      c.vscale[cb * G + i] = vs[i];
      c.vzero[cb * G + i] = vz[i];
    }
  } else if (bx == n) {
    const uint16_t* rk = reinterpret_cast<const uint16_t*>(img + L.rk);
    const uint16_t* rv = reinterpret_cast<const uint16_t*>(img + L.rv);
    for (int i = tid; i < n_res * D; i += blockDim.x) {
      const int t = i / D, ch = i % D;
      c.kres[((size_t)unit * SLOTS + t) * D + ch] = __bfloat16_as_ushort(__float2bfloat16_rn(__half2float(__ushort_as_half(rk[i]))));
      c.vres[((size_t)unit * D + ch) * SLOTS + t] = __bfloat16_as_ushort(__float2bfloat16_rn(__half2float(__ushort_as_half(rv[i]))));
    }
    if (tid == 0) {
      const int b = unit / c.Hkv;
      c.n_chunks[b] = n;
      c.res_start[b] = 0;
      c.res_len[b] = n_res;
    }
  } else {
    const uint16_t* S = reinterpret_cast<const uint16_t*>(img + L.S);
    const uint16_t* P = reinterpret_cast<const uint16_t*>(img + L.P);
    for (int i = (bx - n - 1) * blockDim.x + tid; i < D * RANK + RANK; i += (gridDim.x - n - 1) * blockDim.x) {
      if (i < D * RANK) c.S[(size_t)unit * D * RANK + i] = rank ? __half2float(__ushort_as_half(S[i])) : 0.f;
      else c.P[(size_t)unit * RANK + i - D * RANK] = rank ? __half2float(__ushort_as_half(P[i - D * RANK])) : 0.f;
    }
  }
}

// ---------------------------------------------------------------------------
// Prefill flush with the adapter-state update on the 5th-generation tensor
// cores (tcgen05), cache.py:132-158, in two kernels:
//   quant_kernel (one CTA per chunk): K1 keys, channel-wise codes (fp64 decisions,
//       bit-exact); K2 values, FWHT + token-wise codes; the packed words and fp16
//       metadata go to the cache, and the state kernel's operands to a scratch:
//       k_err = k - k_hat as the A_phi tile image (fp16 hi / lo, 128 B swizzle), the
//       value codes as an fp16 tile image and the fp32 value (scale, zero) per token.
//   flush_tc_kernel (one CTA per (unit, feature half h, chunk range)): W_h (the 128
//       features of W1k or W2k, fp16 hi / lo) resident in shared memory; per chunk
//       phi Z = k_err W_h (3 passes hi.hi + hi.lo + lo.hi, M = 128 tokens, N = 128, f32 in
//       TMEM), row softmax (feature_map, adapter.py:80-88) -> s 2^e Phi, and since
//       v_q = s (code - 3/2) + z' (z' the row midpoint):
//       S^T[c][f] += sum_t (code - 3/2)[t][c] 2^-e (s 2^e Phi)[t][f]  (2 passes, exact codes),
//       with P[f] = sum_t Phi[t][f] and (z'^T Phi)[f] reduced in registers and added at the
//       end.  The next chunk's A_phi image streams in while the softmax and S GEMM run.
constexpr int FT_THREADS = 256;
constexpr int FT_TILE = 32768;              // [128][128] fp16 tile
// TMEM columns: phi of even passes, S (half 0), S (half 1 of a two-halves CTA), phi of odd passes
constexpr uint32_t FT_COL_PHI = 0, FT_COL_S = 128, FT_COL_PHI1 = 384, FT_TMEM2 = 512;
constexpr uint32_t FT_IDESC_PHI = (1u << 4) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) | (8u << 24);

struct FtSmem {
  uint8_t w[2][FT_TILE];     // W_h hi / lo: B of the phi GEMM, [K = channel][N = feature]
  uint8_t a[2][FT_TILE];     // A_phi hi / lo: k_err [M = token][K = channel] (128 B swizzle)
  uint8_t cv[FT_TILE];       // value codes (exact fp16): A of the S GEMM, [M = channel][K = token]
  uint8_t ps[2][FT_TILE];    // s' Phi hi / lo: B of the S GEMM, [K = token][N = feature]
  float2 vsz[G];             // value (scale, zero) per token
  float red[2][G];           // softmax row max / sum of the two 64-feature halves
  uint64_t mphi, ms, mc;     // phi GEMM done, S GEMM done, code tile + (s, z) landed
  uint64_t ma[2];            // A_phi hi, lo landed
  uint32_t tbase;
};

// Value codes [token][channel] with an XOR swizzle on channel bits 2-4 (groups of 4
// channels stay contiguous): conflict-free packing reads.
__device__ __forceinline__ int vsw(int t, int ch) { return t * D + (ch ^ (((t ^ (t >> 3)) & 7) << 2)); }
__device__ __forceinline__ uint32_t pack_v_word_sw(const uint8_t* codes, int wi) {  // pack_v_word on vsw
  const int i = wi & 7, lane = (wi >> 3) & 31, w = wi >> 8;
  const int g = lane >> 2, t0 = lane & 3, mt = i >> 2, p = i & 3;
  const int toff[4] = {0, 1, 4, 5};
  uint32_t word = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = 32 * w + 8 * t0 + 2 * mt + toff[q];
      word |= (uint32_t)codes[vsw(t, 32 * p + 8 * j + g)] << (8 * q + 2 * j);
    }
  return word;
}
__device__ __forceinline__ int ft_off(int mn, int k) {  // byte offset of element (mn, k) in an MN-major tile
  return (mn & 7) * 2 + (k & 7) * 16 + (mn >> 3) * 2048 + (k >> 3) * 128;
}
__device__ __forceinline__ void ft_hilo(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}
// P / z'^T Phi on the tensor cores (legacy warp MMA): D[r][f] = sum_t A[r][t] B[t][f] with B =
// s' Phi hi / lo (the S GEMM's B tile) and the 4 nonzero rows of A = 2^10 / s'_t and 2^10 z'_t / s'_t
// as fp16 hi / lo, so P = (D0 + D1) 2^-10 and z'^T Phi = (D2 + D3) 2^-10 (a lane reduce-scatter of
// 2 x 64 values per token thread cost ~1.3 K cycles per pass)
__device__ __forceinline__ void ft_ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ft_mma16816(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
#ifndef KVLC_EXP_FMA
#define KVLC_EXP_FMA 3  // of every 8 softmax exponentials on the FMA pipe
#endif
// 2^x for x <= 0 on the FMA pipe (round-to-nearest integer split, degree-6 Taylor of 2^f on
// |f| <= 1/2: ~1.2e-7 relative, like ex2.approx; x < -125 gives ~2^-125 instead of ex2.ftz's 0)
__device__ __forceinline__ float ft_exp2_fma(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: the integer part in the low mantissa bits
  const float f = x - (t - 12582912.f);
  float p = 1.5403530e-4f;
  p = fmaf(p, f, 1.3333558e-3f);
  p = fmaf(p, f, 9.6181291e-3f);
  p = fmaf(p, f, 5.5504109e-2f);
  p = fmaf(p, f, 2.4022651e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
// ft_hilo of two values with packed conversions (the same bits: each half is rounded to nearest)
__device__ __forceinline__ void ft_hilo2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ uint64_t ft_desc(const void* p) { return tc::bdesc(tc::smem_u32(p)); }

// A tiles (A_phi = k_err [M = token][K = channel], A_S = Phi^T [M = feature][K = token]) in the
// MN-major SWIZZLE_128B canonical layout: a 128 B row holds 64 MN elements of one K, 8 K rows
// form a 1024 B atom whose 16 B chunks are XOR-ed with the row, K groups of 8 follow at 1024 B,
// the second 64-wide MN block at 16 KB.  A warp storing one K for 128 MN (K1') or 8 MN for 32
// K (softmax) hits every bank once per wavefront; the no-swizzle layout put one K of all
// 8-wide MN groups in the same 4 banks (16-way conflicts).
#ifndef KVLC_FT_LBO
#define KVLC_FT_LBO 16384
#endif
#ifndef KVLC_FT_SBO
#define KVLC_FT_SBO 1024
#endif
__device__ __forceinline__ int ft_off_a(int mn, int k) {
  return (mn >> 6) * 16384 + (k >> 3) * 1024 + (k & 7) * 128 + ((((mn & 63) >> 3) ^ (k & 7)) << 4) + (mn & 7) * 2;
}
__device__ __forceinline__ uint64_t ft_desc_a(const void* p) {
  return (uint64_t)((tc::smem_u32(p) >> 4) & 0x3fff) | ((uint64_t)(KVLC_FT_LBO >> 4) << 16) |
         ((uint64_t)(KVLC_FT_SBO >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
constexpr int FT_A_KSTEP = 2048 >> 4;  // descriptor advance per K = 16 step (two 8-row groups)

// 3 passes (hi*hi, hi*lo, lo*hi) of a K = 128 contraction: 24 MMAs, one elected lane.
// `late` (optional): an mbarrier (phase `parity`) guarding the operand first used by pass
// `late_pass` (a lo tile still in flight while the earlier passes run).
__device__ __forceinline__ void ft_gemm(uint32_t d, const uint8_t (*a)[FT_TILE], const uint8_t* b0, const uint8_t* b1,
                                        uint32_t idesc, bool accumulate, uint64_t* late = nullptr,
                                        uint32_t parity = 0, int late_pass = 3) {
  const uint64_t ah = ft_desc_a(a[0]), al = ft_desc_a(a[1]), bh = ft_desc(b0), bl = ft_desc(b1);
  const uint64_t pa[3] = {ah, ah, al}, pb[3] = {bh, bl, bh};
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    if (late && p == late_pass) {
      tc::mbar_wait(late, parity);
      tc::fence_after_sync();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t acc = (accumulate || p > 0 || j > 0) ? 1u : 0u;
      asm volatile(
          "{\n.reg .pred q, e;\nsetp.ne.b32 q, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n}\n" ::"r"(d),
          "l"(pa[p] + FT_A_KSTEP * j), "l"(pb[p] + 16 * j), "r"(idesc), "r"(acc)
          : "memory");
    }
  }
}

// Prefill quantization (K1 + K2) at one chunk per CTA: code decisions, FWHT,
// packed words, fp16 metadata into the cache; fp32 scale / zero and the value
// codes (bytes) into a scratch the tensor-core state kernel reconstructs k_err
// and v_q from (cache.py:141-154).
// W1k / W2k (fp32 [Hkv][128][128]) -> fp16 hi / lo B tiles of the phi GEMM,
// [kvh][half][hi, lo][FT_TILE]: element (k = channel, n = feature); block x of 16 per (kvh, h).
__device__ __forceinline__ void prep_wtiles_block(const kvlc_adapter& ad, int x, int kvh, int h, uint8_t* out) {
  const float* W = (h == 0 ? ad.w1k : ad.w2k) + (size_t)kvh * D * HALF;
  uint8_t* hi = out + ((size_t)kvh * 2 + h) * 2 * FT_TILE;
  uint8_t* lo = hi + FT_TILE;
  for (int i = x * 256 + (int)threadIdx.x; i < D * HALF; i += 16 * 256) {
    const int ch = i / HALF, f = i % HALF;
    __half xh, yl;
    ft_hilo(__ldg(W + i), xh, yl);
    *reinterpret_cast<__half*>(hi + ft_off(f, ch)) = xh;
    *reinterpret_cast<__half*>(lo + ft_off(f, ch)) = yl;
  }
}
constexpr int VT_LD = D + 2;  // staged ring values: row stride (2-way store conflicts at most)
struct QkSmem {
  uint8_t codes[G * D];  // value codes [token][channel] (swizzled, vsw)
  double2 kpar[D];
  float4 kparf[D];
  union {
    uint16_t vt[G / 2][VT_LD];  // a value CTA's ring tokens, token-major (vsplit >= 2)
    uint16_t vp[G][D];          // a prefill chunk's value rows (cp.async during K1)
  };
  double dv[FT_THREADS / 32][D];  // per warp: the token of a dense re-evaluation, fp64
};
#ifdef KVLC_TRACE
__device__ long long g_qtrace[16][128][4];  // quant CTA (0, unit, z): globaltimer start, K1 done, end; SM id
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define QT_STAMP(i)                                                                              \
  do {                                                                                           \
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.z < 16 && blockIdx.y < 128) {            \
      g_qtrace[blockIdx.z][blockIdx.y][i] = gtimer();                                            \
      if (i == 0) {                                                                              \
        unsigned smid;                                                                           \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                                        \
        g_qtrace[blockIdx.z][blockIdx.y][3] = smid;                                              \
      }                                                                                          \
    }                                                                                            \
  } while (0)
// V CTA z = 1, warp 0: per token iteration end time and the fallback level taken (0 fast, 1 fp64 FWHT, 2 dense)
__device__ long long g_qtok[128][24][2];
#define QT_TOK(ti, lvl)                                                                           \
  do {                                                                                            \
    if (lane == 0 && warp == 0 && blockIdx.x == 0 && blockIdx.z == 1 && blockIdx.y < 128 && (ti) < 24) { \
      g_qtok[blockIdx.y][ti][0] = gtimer();                                                       \
      g_qtok[blockIdx.y][ti][1] = (lvl);                                                          \
    }                                                                                             \
  } while (0)
#else
#define QT_STAMP(i) do {} while (0)
#define QT_TOK(ti, lvl) do {} while (0)
#endif
#ifndef KVLC_QK_MINB
#define KVLC_QK_MINB 3  // 3 CTAs per SM (80 registers, 84 B spills) measured 2 % faster than 2
#endif
__global__ void __launch_bounds__(FT_THREADS, KVLC_QK_MINB) quant_kernel(const FlushArgs a, const SeqInfo seq) {
  extern __shared__ __align__(16) uint8_t qk_raw[];  // QkSmem (60 KB: dynamic)
  QkSmem& sm = *reinterpret_cast<QkSmem*>(qk_raw);
  const kvlc_cache& c = a.c;
  const int unit = blockIdx.y, ci = blockIdx.x;
  const int b = unit / c.Hkv;
  if (a.prep_n) {  // the state kernel's W tiles (16 blocks per (kvh, half)) over the first CTAs
    const int lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    for (int p = lin; p < a.prep_n; p += nblk) prep_wtiles_block(a.ad, p % 16, (p / 16) % c.Hkv, p / (16 * c.Hkv), a.wtiles);
  }
  if (ci >= seq.nflush[b]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool writer = true;
  QT_STAMP(0);
  // prefill: chunk ci of the sequence's tokens; ring (decode-time flush): the oldest G slots of
  // the residual ring into the sequence's next chunk (cache.py:132-147)
  const int64_t tok0 = a.ring ? (int64_t)c.res_start[b] + (int64_t)ci * G : (int64_t)ci * G;
  const uint16_t* K = a.ksrc + unit * a.k_unit + tok0 * a.k_t;
  const uint16_t* V = a.vsrc + unit * a.v_unit + tok0 * a.v_t;
  const size_t cb = (size_t)unit * c.max_chunks + (a.ring ? c.n_chunks[b] + ci : ci);
  // 4 channels 4 lane .. 4 lane + 3 of value row t (contiguous, or the ring's channel-major layout)
  auto ldv = [&](int t) -> uint2 {
    if (a.v_c == 1) return __ldg(reinterpret_cast<const uint2*>(V + (size_t)t * a.v_t + lane * 4));
    const uint16_t* p = V + (size_t)t * a.v_t + (size_t)(lane * 4) * a.v_c;
    return make_uint2((uint32_t)__ldg(p) | ((uint32_t)__ldg(p + a.v_c) << 16),
                      (uint32_t)__ldg(p + 2 * a.v_c) | ((uint32_t)__ldg(p + 3 * a.v_c) << 16));
  };
  const size_t slot = (size_t)unit * a.slot_stride + ci;
  const int zpart = blockIdx.z;
  // a prefill chunk's value rows (contiguous token rows) are copied into shared memory while K1
  // runs: K2 then reads its tokens with one 8-B load per lane, no address math or register ring
  const bool pstaged = a.vsplit == 0 && a.v_c == 1 && (a.v_t & 7) == 0 && (reinterpret_cast<uintptr_t>(V) & 15) == 0;
  if (pstaged) {
    for (int i = tid; i < G * D / 8; i += FT_THREADS)
      tc::cp_async16(&sm.vp[i / (D / 8)][(i % (D / 8)) * 8], V + (size_t)(i / (D / 8)) * a.v_t + (i % (D / 8)) * 8);
    tc::cp_commit();
  }
  if (zpart == 0) {
    // ---- K1: keys, channel-wise.  Warp w: channels 16w..16w+15; lane l: tokens 4l..4l+3
    // (16-B vector loads).  Codes in fp32 with the exact fp64 decision near rounding
    // ties (quantize.py:202-207 bit-exact); the lane also packs the fragment-native
    // K words of its 4 tokens x 16 channels (pack_k_word layout).
    {
      const int ch0 = 16 * warp;
      float x[4][16];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint4* src = reinterpret_cast<const uint4*>(K + (size_t)(4 * lane + r) * D + ch0);
        const uint4 p0 = __ldg(src), p1 = __ldg(src + 1);
        const uint32_t wv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          x[r][2 * e] = __uint_as_float(wv[e] << 16);
          x[r][2 * e + 1] = __uint_as_float(wv[e] & 0xffff0000u);
        }
      }
      // channel min / max over the 128 tokens: reduce-scatter over the lanes
      float mn16[16], mx16[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        mn16[e] = fminf(fminf(x[0][e], x[1][e]), fminf(x[2][e], x[3][e]));
        mx16[e] = fmaxf(fmaxf(x[0][e], x[1][e]), fmaxf(x[2][e], x[3][e]));
      }
      int n = 16;
#pragma unroll
      for (int sft = 16; sft >= 2; sft >>= 1) {
        const bool up = lane & sft;
        n >>= 1;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < n) {
            const float sa = up ? mn16[e] : mn16[e + n], ka = up ? mn16[e + n] : mn16[e];
            const float sb = up ? mx16[e] : mx16[e + n], kb = up ? mx16[e + n] : mx16[e];
            mn16[e] = fminf(ka, __shfl_xor_sync(0xffffffffu, sa, sft));
            mx16[e] = fmaxf(kb, __shfl_xor_sync(0xffffffffu, sb, sft));
          }
        }
      }
      mn16[0] = fminf(mn16[0], __shfl_xor_sync(0xffffffffu, mn16[0], 1));
      mx16[0] = fmaxf(mx16[0], __shfl_xor_sync(0xffffffffu, mx16[0], 1));
      // lane pair (2e', 2e'+1) owns channel ch0 + e(l): bits of l >> 1 select the kept halves
      const int own = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
      if ((lane & 1) == 0) {
        const double mn = (double)mn16[0], mx = (double)mx16[0];
        const double scale = __ddiv_rn(__dsub_rn(mx, mn), 3.0);
        sm.kpar[ch0 + own] = make_double2(mn, scale);
        sm.kparf[ch0 + own] = make_float4((float)mn, (float)scale, scale > 0.0 ? (float)(1.0 / scale) : 0.f, 0.f);
        if (writer) {
          c.kscale[cb * D + ch0 + own] = __half_as_ushort(__double2half(scale));
          c.kzero[cb * D + ch0 + own] = __half_as_ushort(__double2half(mn));
        }
      }
      __syncwarp();
      uint32_t cw[4] = {0u, 0u, 0u, 0u};  // K words t0 = 0..3 of this lane's tokens
      uint8_t* aimg = a.aimg + slot * 2 * FT_TILE;
      // elements near a rounding tie (bit 4e + r) are re-decided after the loop: an inlined
      // fp64 division per element made the unrolled loop ~60 KB of SASS (instruction-fetch
      // stalls, the key CTA of a ring flush took ~35 us)
      uint64_t tie = 0;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float4 pf = sm.kparf[ch0 + e];
        const float mnf = pf.x, scf = pf.y, invf = pf.z;
        float kerr[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          uint32_t code = 0u;
          if (scf > 0.f) {
            const float q = (x[r][e] - mnf) * invf;
            const float fr = q - floorf(q);
            tie |= (uint64_t)(fabsf(fr - 0.5f) < 1e-5f) << (4 * e + r);
            code = (uint32_t)fminf(fmaxf(rintf(q), 0.f), 3.f);
          }
          // byte q of word t0 holds channel 16kt + 2t0 + {0,8,1,9}[q]; bit pair r holds token 4l + r
          const int t0 = (e & 7) >> 1, qb = ((e & 1) << 1) | (e >> 3);
          cw[t0] |= code << (8 * qb + 2 * r);
          // k_err = k - (s code + z) (cache.py:153), stored as an fp16 hi / lo pair
          kerr[r] = x[r][e] - fmaf((float)code, scf, mnf);
        }
        // A_phi image element (tokens 4l .. 4l+3, channel ch0 + e): 8 contiguous bytes
        uint2 ehi, elo;
        ft_hilo2(kerr[0], kerr[1], ehi.x, elo.x);
        ft_hilo2(kerr[2], kerr[3], ehi.y, elo.y);
        const int off = ft_off_a(4 * lane, ch0 + e);
        *reinterpret_cast<uint2*>(aimg + off) = ehi;
        *reinterpret_cast<uint2*>(aimg + FT_TILE + off) = elo;
      }
      while (tie) {  // the exact fp64 decision (quantize.py:202-207) for the near-tie elements
        const int bit = __ffsll((long long)tie) - 1;
        tie &= tie - 1;
        const int e = bit >> 2, r = bit & 3;
        const float xv = bf2f(K[(size_t)(4 * lane + r) * D + ch0 + e]);
        const double2 pr = sm.kpar[ch0 + e];
        const uint32_t code = code_of((double)xv, pr.x, pr.y, 3);
        const int t0 = (e & 7) >> 1, sh = 8 * (((e & 1) << 1) | (e >> 3)) + 2 * r;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k == t0) cw[k] = (cw[k] & ~(3u << sh)) | (code << sh);
        const float4 pf = sm.kparf[ch0 + e];
        __half hi, lo;
        ft_hilo(xv - fmaf((float)code, pf.y, pf.x), hi, lo);
        const int off = ft_off_a(4 * lane, ch0 + e) + 2 * r;
        *reinterpret_cast<__half*>(aimg + off) = hi;
        *reinterpret_cast<__half*>(aimg + FT_TILE + off) = lo;
      }
      if (writer) {
        const int wt = lane >> 3, g = lane & 7;  // tokens 32 wt + 4 g + r
#pragma unroll
        for (int t0 = 0; t0 < 4; ++t0) c.kcodes[cb * 1024 + ((wt * 32 + 4 * g + t0) * 8 + warp)] = frag_store(cw[t0]);
      }
    }
  }
  QT_STAMP(1);
  // token range of K2: the whole chunk, or 32-token slice zpart - 1
  const int t_lo = a.vsplit ? (zpart - 1) * (G / a.vsplit) : 0;
  const int ntok_w = a.vsplit ? G / a.vsplit / (FT_THREADS / 32) : G / (FT_THREADS / 32);  // per warp
  if (a.vsplit == 0 || zpart > 0) {
    // The ring holds values channel-major ([D][SLOTS], for the decode's residual MMAs): a
    // value CTA of <= 64 tokens stages its slice token-major in shared memory with 16-B loads
    // along the slot axis (per-lane 2-B gathers from 128 channel rows made the value CTAs of a
    // decode-time flush take ~20 us)
    const int ntok = a.vsplit ? G / a.vsplit : G;
    const bool staged = a.v_c != 1 && a.v_t == 1 && ntok <= G / 2 && ntok % 8 == 0 &&
                        (reinterpret_cast<uintptr_t>(V) & 15) == 0 && (a.v_c & 7) == 0;
    if (pstaged) {
      tc::cp_wait<0>();
      __syncthreads();
    }
    if (staged) {
      const int per_row = ntok / 8;
      for (int i = tid; i < D * per_row; i += FT_THREADS) {
        const int ch = i / per_row, tg = i % per_row;
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(V + (size_t)ch * a.v_c + t_lo + 8 * tg));
        const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) sm.vt[8 * tg + j][ch] = (uint16_t)(wv[j >> 1] >> (16 * (j & 1)));
      }
      __syncthreads();
    }
    // ---- K2: values, FWHT post-rotation (fp32, guarded), token-wise quantization ----
    // The fp32 FWHT differs from the reference's fp64 dense x @ H in the last bits:
    // a token whose quotient lies near a rounding tie or whose scale / zero lies near
    // an fp16 rounding midpoint is re-evaluated in the reference's exact order.
#ifdef KVLC_TRACE
    int n_lvl = 0;
#endif
    // the token loop compiled once per source kind (a runtime `staged` test inside it was
    // if-converted: both load paths issued for every token, ~60 instructions)
    // source kinds: 0 global (register ring), 1 ring values staged (vt), 2 prefill rows staged (vp)
    auto k2_tokens = [&](auto st_c) {
      constexpr int SRC = decltype(st_c)::value;
      constexpr bool ST = SRC != 0;
      auto ldvs = [&](int t) -> uint2 {
        if constexpr (SRC == 1) {
          const uint32_t* p = reinterpret_cast<const uint32_t*>(&sm.vt[t - t_lo][lane * 4]);
          return make_uint2(p[0], p[1]);
        } else if constexpr (SRC == 2) {
          return *reinterpret_cast<const uint2*>(&sm.vp[t][lane * 4]);
        } else {
          return ldv(t);
        }
      };
      // rolling 8-deep register prefetch of this warp's 16 value rows (one 8-B piece per lane)
      constexpr int VPF = 8;
      uint2 vpf[VPF];
  #pragma unroll
      for (int i = 0; i < VPF; ++i)
        if (!ST && i < ntok_w) vpf[i] = ldv(t_lo + warp + 8 * i);
      QT_TOK(0, 0);
  #pragma unroll 1
      for (int ti = 0; ti < ntok_w; ++ti) {
        const int t = t_lo + warp + 8 * ti;
  #ifdef KVLC_TRACE
        int lvl = 0;
        if (ti == 0) n_lvl = 0;
  #endif
        float xf[4];
        {
          uint2 raw;
          if (ST) {
            raw = ldvs(t);
          } else {
            raw = vpf[0];
  #pragma unroll
            for (int i = 0; i < VPF - 1; ++i) vpf[i] = vpf[i + 1];
            if (ti + VPF < ntok_w) vpf[VPF - 1] = ldv(t + 8 * VPF);
          }
          xf[0] = __uint_as_float(raw.x << 16);
          xf[1] = __uint_as_float(raw.x & 0xffff0000u);
          xf[2] = __uint_as_float(raw.y << 16);
          xf[3] = __uint_as_float(raw.y & 0xffff0000u);
        }
        float u0 = xf[0] + xf[1], u1 = xf[0] - xf[1], u2 = xf[2] + xf[3], u3 = xf[2] - xf[3];
        xf[0] = u0 + u2;
        xf[2] = u0 - u2;
        xf[1] = u1 + u3;
        xf[3] = u1 - u3;
  #pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float o = __shfl_xor_sync(0xffffffffu, xf[e], k);
            xf[e] = fmaf(xf[e], (lane & k) ? -1.f : 1.f, o);  // o - x or x + o, one FFMA (exact)
          }
        }
        const float hsf = 0.08838834764831845f;
        // row min / max of the unnormalised transform (scaling by hsf > 0 keeps the order, so
        // mnf = mnu * hsf is bit-identical to the min of the scaled values)
        float mnu = INFINITY, mxu = -INFINITY;
  #pragma unroll
        for (int e = 0; e < 4; ++e) {
          mnu = fminf(mnu, xf[e]);
          mxu = fmaxf(mxu, xf[e]);
          xf[e] *= hsf;
        }
        mnu = warp_min(mnu);
        mxu = warp_max(mxu);
        float mnf = mnu * hsf, mxf = mxu * hsf;
        // Fast path in fp32.  fp32 FWHT error: a few ulps of the token's largest magnitude
        // (ferr); a token is re-evaluated exactly when a quotient lies within qtol of a
        // rounding tie or its zero / scale lies near an fp16 rounding midpoint (the stored
        // metadata is float16 of the reference's fp64 value, cache.py:220-224).
        const float range = mxf - mnf;
        // approximate divisions: invf feeds only the fast-path quotients (error ~1e-7, inside
        // qtol) and the rest are tolerances
        const float scf = range * (1.f / 3.f), invf = range > 0.f ? __fdividef(3.f, range) : 0.f;
        const float ferr = 4e-6f * fmaxf(fabsf(mnf), fabsf(mxf));
        auto near_mid = [](float v, float rel) {
          return __half_as_ushort(__float2half_rn(v * (1.f - rel))) != __half_as_ushort(__float2half_rn(v * (1.f + rel)));
        };
        bool amb = near_mid(mnf, __fdividef(ferr, fmaxf(fabsf(mnf), 1e-30f)) + 2e-7f) ||
                   (range > 0.f && near_mid(scf, __fdividef(2.f * ferr, range) + 2e-7f));
        const float qtol = 1e-4f + 4.f * ferr * invf;
        uint32_t code[4];
  #pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float q = (xf[e] - mnf) * invf;
          amb |= range > 0.f && fabsf(q - floorf(q) - 0.5f) < qtol;
          code[e] = range > 0.f ? (uint32_t)fminf(fmaxf(rintf(q), 0.f), 3.f) : 0u;
        }
        // the state kernel's fp32 (s, z') of v_q = s code + z: from the unnormalised min / max in
        // fp64, each rounded once.  fp32(1/sqrt(128)) is 1.7e-8 low and fp32(1/3) 3e-8 high, and
        // z' = z + 3/2 s enters S as the same-signed rank-1 term sum_t z'_t Phi_t for every
        // token: a fixed relative bias of the per-token (s, z') grew the S error ~ n / sqrt(n)
        // (4.0e-6 at 8k, 1.9e-5 at 131k tokens, 97 % of it channel-constant; tools/s_error_diag.py)
        const double hsd = 0.088388347648318440550;  // 1 / sqrt(128)
        float vsc = (float)(((double)mxu - (double)mnu) * (hsd / 3.0));
        float vmid = (float)(0.5 * ((double)mnu + (double)mxu) * hsd);
        uint16_t meta_s = __half_as_ushort(__float2half_rn(scf)), meta_z = __half_as_ushort(__float2half_rn(mnf));
  #ifdef KVLC_FORCE_DENSE
        amb = true;
  #endif
        if (__any_sync(0xffffffffu, amb)) {
  #ifdef KVLC_TRACE
          lvl = 1;
  #endif
          // fp64 FWHT: agrees with the dense fp64 x @ H to an ulp
          const double hs = 1.0 / sqrt((double)D);
          double x[4], y[4];
          {
            const uint2 raw = ldvs(t);
            y[0] = (double)__uint_as_float(raw.x << 16);
            y[1] = (double)__uint_as_float(raw.x & 0xffff0000u);
            y[2] = (double)__uint_as_float(raw.y << 16);
            y[3] = (double)__uint_as_float(raw.y & 0xffff0000u);
          }
          double w0 = y[0] + y[1], w1 = y[0] - y[1], w2 = y[2] + y[3], w3 = y[2] - y[3];
          y[0] = w0 + w2;
          y[2] = w0 - w2;
          y[1] = w1 + w3;
          y[3] = w1 - w3;
  #pragma unroll
          for (int k = 1; k < 32; k <<= 1) {
  #pragma unroll
            for (int e = 0; e < 4; ++e) {
              const double o = __shfl_xor_sync(0xffffffffu, y[e], k);
              y[e] = fma(y[e], (lane & k) ? -1.0 : 1.0, o);  // o - x or x + o (exact)
            }
          }
          double mn = INFINITY, mx = -INFINITY;
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            x[e] = y[e] * hs;
            mn = fmin(mn, x[e]);
            mx = fmax(mx, x[e]);
          }
          mn = warp_min_d(mn);
          mx = warp_max_d(mx);
          double scale = __ddiv_rn(__dsub_rn(mx, mn), 3.0);
          double inv = scale > 0.0 ? 1.0 / scale : 0.0;
          bool amb2 = near_half_tie(scale) || near_half_tie(mn);
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const double r = __dsub_rn(x[e], mn) * inv;
            amb2 |= scale > 0.0 && fabs(r - floor(r) - 0.5) < 1e-9;
          }
  #ifdef KVLC_FORCE_DENSE  // timing probe: every ambiguous token takes the dense path
          amb2 = true;
  #endif
          if (__any_sync(0xffffffffu, amb2)) {  // a genuine tie: the reference's dense x @ H order
  #ifdef KVLC_TRACE
            lvl = 2;
  #endif
            mn = INFINITY;
            mx = -INFINITY;
            // the lane's 4 channel chains interleaved (each chain keeps its j order: the same
            // sums as one chain after another, ~4x less latency; the serial form cost ~19 us)
            // H[j][4 lane + e] = (-1)^(popc(J & lane) + popc(r & e)) hs for j = 4 J + r
            {
              const uint2 rw = ldvs(t);  // the token in fp64 in shared memory (one conversion per value)
              double4* d4 = reinterpret_cast<double4*>(&sm.dv[warp][4 * lane]);
              *d4 = make_double4((double)__uint_as_float(rw.x << 16), (double)__uint_as_float(rw.x & 0xffff0000u),
                                 (double)__uint_as_float(rw.y << 16), (double)__uint_as_float(rw.y & 0xffff0000u));
              __syncwarp();
            }
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
  #pragma unroll 2
            for (int J = 0; J < D / 4; ++J) {
              const double sg = (__popc((unsigned)(J & lane)) & 1) ? -hs : hs;
  #pragma unroll
              for (int r = 0; r < 4; ++r) {
                const double v = sm.dv[warp][4 * J + r];
  #pragma unroll
                for (int e = 0; e < 4; ++e) acc[e] = fma(v, (__popc(r & e) & 1) ? -sg : sg, acc[e]);
              }
            }
            __syncwarp();
  #pragma unroll
            for (int e = 0; e < 4; ++e) {
              x[e] = acc[e];
              mn = fmin(mn, acc[e]);
              mx = fmax(mx, acc[e]);
            }
            mn = warp_min_d(mn);
            mx = warp_max_d(mx);
            scale = __ddiv_rn(__dsub_rn(mx, mn), 3.0);
            inv = scale > 0.0 ? 1.0 / scale : 0.0;
          }
  #pragma unroll
          for (int e = 0; e < 4; ++e) code[e] = code2(x[e], mn, scale, inv);
          vsc = (float)scale;
          vmid = (float)(mn + 1.5 * scale);
          meta_s = __half_as_ushort(__double2half(scale));
          meta_z = __half_as_ushort(__double2half(mn));
        }
        const uint32_t cword = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
        *reinterpret_cast<uint32_t*>(sm.codes + vsw(t, lane * 4)) = cword;
        {  // codes -> the state kernel's A tile (channels 4l .. 4l+3, token t).  v_q = s code + z
           // (cache.py:154) is applied there as S = ((code - 3/2) 2^-e)^T (s 2^e Phi) + 1 (z'^T Phi),
           // z' = z + 3/2 s the row midpoint: centred codes keep the two terms from cancelling
           // (z alone is ~ -2 for N(0,1) rows, S ~ 0.5), the per-token power of two 2^e puts
           // s 2^e in [2^10, 2^11) so the fp16 hi / lo split of s 2^e Phi stays out of the
           // subnormal range, and (code - 3/2) 2^-e is exact in fp16
          // frexpf exponent from the bits (a subnormal vsc clamps to e = 22 either way)
          const int ex = (int)((__float_as_uint(vsc > 0.f ? vsc : 1.f) >> 23) & 0xffu) - 126;
          const int e = min(max(11 - ex, -14), 22);
          const float cs = __int_as_float((127 - e) << 23);  // 2^-e
          auto hc = [&](uint32_t cd) { return (uint32_t)__half_as_ushort(__float2half_rn(((float)cd - 1.5f) * cs)); };
          *reinterpret_cast<uint2*>(a.cimg + slot * FT_TILE + ft_off(4 * lane, t)) =
              make_uint2(hc(code[0]) | (hc(code[1]) << 16), hc(code[2]) | (hc(code[3]) << 16));
          // a constant row (s = 0, codes 0) is stored as s = 1, z' = z + 3/2: the same
          // (code - 3/2) s + z' = z, and the state kernel's 1 / s' exists
          if (lane == 0)
            a.vsz[slot * G + t] = vsc > 0.f ? make_float2(vsc * __int_as_float((127 + e) << 23), vmid)
                                            : make_float2(__int_as_float((127 + e) << 23), vmid + 1.5f);
        }
        if (writer && lane == 0) {
          c.vscale[cb * G + t] = meta_s;
          c.vzero[cb * G + t] = meta_z;
        }
        QT_TOK(ti + 1, lvl);
  #ifdef KVLC_TRACE
        n_lvl += lvl == 1 ? 1 : lvl == 2 ? 256 : 0;
  #endif
      }
    };
    if (staged)
      k2_tokens(std::integral_constant<int, 1>{});
    else if (pstaged)
      k2_tokens(std::integral_constant<int, 2>{});
    else
      k2_tokens(std::integral_constant<int, 0>{});
#ifdef KVLC_TRACE
    if (lane == 0 && blockIdx.x == 0 && blockIdx.z == 1 && blockIdx.y < 128) {
      g_qtok[blockIdx.y][9 + warp][0] = gtimer();
      g_qtok[blockIdx.y][9 + warp][1] = n_lvl;
    }
#endif
    __syncthreads();
#ifdef KVLC_TRACE
    if (tid == 0 && blockIdx.x == 0 && blockIdx.z == 1 && blockIdx.y < 128) g_qtok[blockIdx.y][17][0] = gtimer();
#endif
    // V words of the CTA's slices (a word covers tokens of one 32-token slice: 256 words each)
    const int w_lo = a.vsplit ? (zpart - 1) * (1024 / a.vsplit) : 0, w_hi = a.vsplit ? w_lo + 1024 / a.vsplit : 1024;
    for (int wi = w_lo + tid; wi < w_hi; wi += FT_THREADS) c.vcodes[cb * 1024 + wi] = frag_store(pack_v_word_sw(sm.codes, wi));
  }
  QT_STAMP(2);
#ifdef KVLC_TRACE
  if (tid == 0 && blockIdx.x == 0 && blockIdx.z == 1 && blockIdx.y < 128) g_qtok[blockIdx.y][18][0] = gtimer();
#endif
}

#ifdef KVLC_TRACE
__device__ long long g_ftrace[2][40][10];  // CTA (0, 0, h): per chunk clock64 at phase boundaries (thread 0)
#define FT_STAMP(i)                                                                            \
  do {                                                                                         \
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && it < 40) g_ftrace[h0 + hp][it][i] = clock64(); \
  } while (0)
// kernel phases of CTA (0, 0, h0) in slot 39: entry, setup done, chunk loop done, drain done
#define FT_PHASE(i) \
  do { if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_ftrace[h0][39][i] = clock64(); } while (0)
// drain steps of pass hp in slot 38: start, P done, tile written, rows written
#define FT_DRAIN(i) \
  do { if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_ftrace[h0 + hp][38][i] = clock64(); } while (0)
#else
#define FT_DRAIN(i) do { } while (0)
#define FT_STAMP(i) \
  do {              \
  } while (0)
#define FT_PHASE(i) do { } while (0)
#endif

// The chunk's operand images (written by quant_kernel) into the shared-memory tiles.
// (hi and lo on separate barriers: the GEMMs' first two passes need only the hi tiles)
__device__ __forceinline__ void ft_load_a(FtSmem& sm, const FlushArgs& a, size_t slot) {
  const uint8_t* src = a.aimg + slot * 2 * FT_TILE;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    tc::mbar_expect_tx(&sm.ma[i], FT_TILE);
    tc::bulk_g2s(sm.a[i], src + i * FT_TILE, FT_TILE, &sm.ma[i]);
  }
}
__device__ __forceinline__ void ft_load_c(FtSmem& sm, const FlushArgs& a, size_t slot) {
  tc::mbar_expect_tx(&sm.mc, FT_TILE + G * sizeof(float2));
  tc::bulk_g2s(sm.cv, a.cimg + slot * FT_TILE, FT_TILE, &sm.mc);
  tc::bulk_g2s(sm.vsz, a.vsz + slot * G, G * sizeof(float2), &sm.mc);
}

// S GEMM (D^T[c][f] += sum_t code[t][c] (s' Phi)[t][f]): 2 passes (codes are exact in fp16).
__device__ __forceinline__ void ft_gemm_s(uint32_t d, const uint8_t* cv, const uint8_t* b0, const uint8_t* b1,
                                          bool accumulate) {
  const uint64_t ac = ft_desc(cv), pb[2] = {ft_desc(b0), ft_desc(b1)};
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t acc = (accumulate || p > 0 || j > 0) ? 1u : 0u;
      asm volatile(
          "{\n.reg .pred q, e;\nsetp.ne.b32 q, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n}\n" ::"r"(d),
          "l"(ac + 16 * j), "l"(pb[p] + 16 * j), "r"(FT_IDESC_PHI), "r"(acc)
          : "memory");
    }
}

__global__ void __launch_bounds__(FT_THREADS, 1) flush_tc_kernel(const FlushArgs a, const SeqInfo seq,
                                                                 const uint8_t* __restrict__ wtiles) {
  extern __shared__ __align__(1024) uint8_t ft_raw[];
  FtSmem& sm = *reinterpret_cast<FtSmem*>(ft_raw);
  const kvlc_cache& c = a.c;
  const int unit = blockIdx.y, split = blockIdx.x;
  // feature halves of this CTA: blockIdx.z, or both in turn (a.both: one chunk per CTA, the
  // decode-time ring flush; 128 CTAs in one wave instead of 256 in two)
  const int h0 = a.both ? 0 : (int)blockIdx.z, npass = a.both ? 2 : 1;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nf = seq.nflush[b];
  const int c_lo = split * a.cpc, c_hi = min(nf, c_lo + a.cpc);
  if (a.finalize && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) append_finalize(c, seq);
  if (c_lo >= c_hi) return;
  const size_t slot0 = (size_t)unit * a.slot_stride;
  FT_PHASE(0);
  if (!a.s_out && tid <= D) {  // the drain's read-modify-write rows (S, P: this CTA's halves) into L2 now
    const float* row = (tid < D ? c.S + ((size_t)unit * D + tid) * RANK : c.P + (size_t)unit * RANK) + h0 * HALF;
    if (npass == 2)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], 1024;\n" ::"l"(row) : "memory");
    else
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;\n" ::"l"(row) : "memory");
  }

  // resident W_h tiles (prepared by quant_kernel), TMEM, barriers, first images
  {
    const uint4* src = reinterpret_cast<const uint4*>(wtiles + ((size_t)kvh * 2 + h0) * 2 * FT_TILE);
    uint4* dst = reinterpret_cast<uint4*>(sm.w[0]);
    for (int i = tid; i < 2 * FT_TILE / 16; i += FT_THREADS) tc::cp_async16(dst + i, src + i);
    tc::cp_commit();
  }
  if (warp == 0) tc::tmem_alloc(&sm.tbase, FT_TMEM2);
  if (tid == 0) {
    tc::mbar_init(&sm.mphi, 1);
    tc::mbar_init(&sm.ms, 1);
    tc::mbar_init(&sm.mc, 1);
    tc::mbar_init(&sm.ma[0], 1);
    tc::mbar_init(&sm.ma[1], 1);
    tc::mbar_fence_init();
    ft_load_a(sm, a, slot0 + c_lo);
    ft_load_c(sm, a, slot0 + c_lo);
  }
  tc::cp_wait<0>();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if ((tc::smem_u32(sm.a[0]) & 1023u) != 0) __trap();  // swizzle atoms must be 1024 B aligned
  const uint32_t tb = sm.tbase;
  const uint32_t lane_addr = tb + ((uint32_t)(32 * (warp & 3)) << 16);
  const int part = warp >> 2;
  // P[f] = sum_t phi[t][f], Z[f] = sum_t z_t phi[t][f] for this warp's 32 token rows:
  // lane owns features 64 part + 2 lane + {0, 1} (reduce-scatter order)
  // MMA accumulators of the P / z'^T Phi rows per half (pz0, pz1) and n-tile (registers: the
  // half is selected by a branch, not an index)
  float pz0[2][4], pz1[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) pz0[j][e] = pz1[j][e] = 0.f;
  FT_PHASE(1);
  // pass pi: chunk ci = c_lo + pi / npass, half h0 + hp (hp = pi % npass).  Barrier phases: the
  // A / code tiles complete once per chunk (ic), the phi / S GEMMs once per pass (it = pi)
  // phi GEMM of pass q: Z = k_err W_h into the pass's phi columns (hi.hi, hi.lo once A hi has
  // landed, lo.hi after A lo).  Pass 0's is issued here; pass q + 1's right after pass q's S GEMM,
  // so it runs on the tensor cores while pass q's warps finish (P / Z MMAs, code tile) and is done
  // when pass q + 1's softmax starts (r02: phi issue + wait was 2.3 K of 7.8 K cycles per pass)
  const int npi = npass * (c_hi - c_lo);
  auto issue_phi = [&](int q) {
    const int qh = q % npass, qc = q / npass;
    if (qh == 0) tc::mbar_wait(&sm.ma[0], (uint32_t)qc & 1u);
    tc::fence_after_sync();
    ft_gemm(tb + ((q & 1) ? FT_COL_PHI1 : FT_COL_PHI), sm.a, sm.w[0], sm.w[1], FT_IDESC_PHI, false,
            qh == 0 ? &sm.ma[1] : nullptr, (uint32_t)qc & 1u, 2);
    tc::mma_commit_w(&sm.mphi);
  };
  if (warp == FT_THREADS / 32 - 1) issue_phi(0);
  for (int pi = 0; pi < npi; ++pi) {
    const int hp = pi % npass, ic = pi / npass, ci = c_lo + ic, it = pi;
    const uint32_t col_phi = (pi & 1) ? FT_COL_PHI1 : FT_COL_PHI;
    FT_STAMP(0);
    FT_STAMP(1);
    tc::mbar_wait(&sm.mphi, (uint32_t)it & 1u);
    tc::fence_after_sync();
    // A_phi consumed by the chunk's last pass: the next chunk's in flight
    if (tid == 0 && hp == npass - 1 && ci + 1 < c_hi) ft_load_a(sm, a, slot0 + ci + 1);
    if (npass == 2 && pi + 1 < npass * (c_hi - c_lo)) {  // the other half's W into the freed W tiles
      const uint4* src = reinterpret_cast<const uint4*>(wtiles + ((size_t)kvh * 2 + (1 - hp)) * 2 * FT_TILE);
      uint4* dst = reinterpret_cast<uint4*>(sm.w[0]);
      for (int i = tid; i < 2 * FT_TILE / 16; i += FT_THREADS) tc::cp_async16(dst + i, src + i);
      tc::cp_commit();
    }
    if (hp == 0) tc::mbar_wait(&sm.mc, (uint32_t)ic & 1u);  // this chunk's codes and (s, z)
    if (it > 0) tc::mbar_wait(&sm.ms, (uint32_t)(it - 1) & 1u);  // the previous S GEMM has read s' Phi
    FT_STAMP(2);

    // ---- softmax of Z (token rows; feature_map, adapter.py:80-88): warps w and w + 4 share TMEM
    // lanes 32 (w & 3) .., 64 feature columns each ----
    {
      const int t = 32 * (warp & 3) + lane;
      float z[64];
      tc::tmem_ld32(lane_addr + col_phi + 64 * part, reinterpret_cast<uint32_t*>(z));
      tc::tmem_ld32(lane_addr + col_phi + 64 * part + 32, reinterpret_cast<uint32_t*>(z) + 32);
      tc::wait_ld();
      FT_STAMP(5);
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // 4 chains (exact: max)
#pragma unroll
      for (int i = 0; i < 64; ++i) m4[i & 3] = fmaxf(m4[i & 3], z[i]);
      float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      sm.red[part][t] = m;
      __syncthreads();
      m = fmaxf(sm.red[0][t], sm.red[1][t]) * 1.4426950408889634f;
      FT_STAMP(6);
      float s4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 partial sums: a 64-deep add chain was latency
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        // 3 of every 8 on the FMA pipe: the MUFU (16 ex2 per clock per SM) bounded this loop
        float e2;
        const float xe = fmaf(z[i], 1.4426950408889634f, -m);
        if ((i & 7) < KVLC_EXP_FMA)
          e2 = ft_exp2_fma(xe);
        else
          asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(xe));
        z[i] = e2;
        s4[i & 3] += e2;
      }
      const float ssum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      __syncthreads();
      sm.red[part][t] = ssum;
      __syncthreads();
      const float inv = 1.f / (sm.red[0][t] + sm.red[1][t]);
      const float2 vz = sm.vsz[t];  // (s 2^e, z'): see quant_kernel
      const float sp = vz.x;
      __syncthreads();  // every thread has read the softmax sums: red takes the P / Z A rows
      if (part == 0) {  // token t: (2^10 / s', 2^10 z' / s') as fp16 hi / lo pairs
        const float is = __frcp_rn(sp) * 1024.f;
        uint32_t hi2, lo2;
        ft_hilo2(is, vz.y * is, hi2, lo2);
        uint32_t* tbl = reinterpret_cast<uint32_t*>(sm.red);
        tbl[t] = __byte_perm(hi2, lo2, 0x5410);        // (inv hi, inv lo)
        tbl[G + t] = __byte_perm(hi2, lo2, 0x7632);    // (z' inv hi, z' inv lo)
      }
      FT_STAMP(7);
      // B of the S GEMM: s' phi, element (token t, feature f); 8 consecutive features = 16 B
#pragma unroll
      for (int f8 = 0; f8 < 64; f8 += 8) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 8; ++e) z[f8 + e] *= inv;
#pragma unroll
        for (int e = 0; e < 4; ++e) ft_hilo2(sp * z[f8 + 2 * e], sp * z[f8 + 2 * e + 1], hi[e], lo[e]);
        *reinterpret_cast<uint4*>(sm.ps[0] + ft_off(64 * part + f8, t)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(sm.ps[1] + ft_off(64 * part + f8, t)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      FT_STAMP(8);
      FT_STAMP(9);
    }
    if (npass == 2) tc::cp_wait<0>();  // the next pass's W (before the barrier below)
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    FT_STAMP(3);
    if (warp == 0) {  // S GEMM: D^T += codes^T (s' Phi), then the next pass's phi GEMM
      tc::fence_after_sync();
      ft_gemm_s(tb + FT_COL_S + 128 * hp, sm.cv, sm.ps[0], sm.ps[1], ic > 0);
      tc::mma_commit_w(&sm.ms);
    }
    // this warp's 16 features (two n-tiles) over the chunk's 128 tokens, into a fresh accumulator
    // added to the running total with round-to-nearest adds (the MMA's truncating accumulation
    // over all chunks drifted P to 2.7e-5 relative at 8k tokens, T3 is 1e-5)
    auto pz_mma = [&](float (&tot)[2][4]) {
      float pz[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) pz[j][0] = pz[j][1] = pz[j][2] = pz[j][3] = 0.f;
      const uint32_t* tbl = reinterpret_cast<const uint32_t*>(sm.red);
      const int g = lane >> 2, t4 = lane & 3, mi = lane >> 3, fb = 16 * warp;
      const uint32_t sel = (g & 1) ? 0x7632u : 0x5410u;  // hi or lo half of the (hi, lo) pairs
      const uint32_t* trow = tbl + ((g >> 1) & 1) * G;
#pragma unroll 2
      for (int k0 = 0; k0 < G; k0 += 16) {
        uint32_t a0 = 0u, a2 = 0u;
        if (g < 4) {
          a0 = __byte_perm(trow[k0 + 2 * t4], trow[k0 + 2 * t4 + 1], sel);
          a2 = __byte_perm(trow[k0 + 2 * t4 + 8], trow[k0 + 2 * t4 + 9], sel);
        }
        const int tok = k0 + (mi & 1) * 8 + (lane & 7), fe = fb + (mi >> 1) * 8;
        uint32_t bh[4], bl[4];
        ft_ldsm_x4_t(tc::smem_u32(sm.ps[0] + ft_off(fe, tok)), bh);
        ft_ldsm_x4_t(tc::smem_u32(sm.ps[1] + ft_off(fe, tok)), bl);
        ft_mma16816(pz[0], a0, a2, bh[0], bh[1]);
        ft_mma16816(pz[1], a0, a2, bh[2], bh[3]);
        ft_mma16816(pz[0], a0, a2, bl[0], bl[1]);
        ft_mma16816(pz[1], a0, a2, bl[2], bl[3]);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) tot[j][e] += pz[j][e];
    };
    if (hp == 0)
      pz_mma(pz0);
    else
      pz_mma(pz1);
    if (warp == 0 && hp == npass - 1 && ci + 1 < c_hi) {  // the next code tile once this one is read
      tc::mbar_wait(&sm.ms, (uint32_t)it & 1u);
      if (lane == 0) ft_load_c(sm, a, slot0 + ci + 1);
      __syncwarp();
    }
    // the A rows (red) and s' Phi reads are done before the next pass writes them.  The last warp
    // only arrives, then issues the next pass's phi GEMM (its issue stalls while the tensor cores
    // drain the S GEMM; the next softmax waits for that GEMM anyway)
    if (warp == FT_THREADS / 32 - 1) {
      asm volatile("bar.arrive 1, %0;\n" ::"r"(FT_THREADS) : "memory");
      if (pi + 1 < npi) issue_phi(pi + 1);
    } else {
      asm volatile("bar.sync 1, %0;\n" ::"r"(FT_THREADS) : "memory");
    }
    FT_STAMP(4);
  }

  // ---- drain: S[c][h*128 + f] = D^T[c][f] + (z^T Phi)[f] (cache.py:155-157), P[h*128 + f] ----
  tc::mbar_wait(&sm.ms, (uint32_t)(npass * (c_hi - c_lo) - 1) & 1u);
  FT_PHASE(2);
  tc::fence_after_sync();
#pragma unroll 1
  for (int hp = 0; hp < npass; ++hp) {
  const int h = h0 + hp;
  if (hp > 0) __syncthreads();  // the previous half's tile / row reads are done
  FT_DRAIN(0);
  float* zf = reinterpret_cast<float*>(sm.ps[0]);  // free now: [P | z'^T Phi][128 features]
  {
    const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float x = hp == 0 ? pz0[nt][e] : pz1[nt][e];
        const float v = x + __shfl_xor_sync(0xffffffffu, x, 4);  // hi + lo rows
        const int f = 16 * warp + 8 * nt + 2 * t4 + e;
        if (g == 0) zf[f] = v * (1.f / 1024.f);
        if (g == 2) zf[G + f] = v * (1.f / 1024.f);
      }
  }
  __syncthreads();
  float* S = a.s_out ? a.s_out + ((size_t)unit * a.splits + split) * D * RANK : c.S + (size_t)unit * D * RANK;
  float* P = a.p_out ? a.p_out + ((size_t)unit * a.splits + split) * RANK : c.P + (size_t)unit * RANK;
  if (tid < HALF) {
    P[h * HALF + tid] += zf[tid];
  }
  FT_DRAIN(1);
  // S rows: TMEM -> a padded shared tile (the W / A tiles are free now) -> coalesced 16-B
  // read-modify-writes of whole S rows with the rank-1 term added (a thread per TMEM row
  // walking its row took ~20 us per CTA: every warp access touched 32 rows, r02
  // tools/trace_flushstep.py)
  {
    constexpr int TLD = 132;  // floats per tile row: 16-B aligned, 4-wavefront float4 stores
    float* tile = reinterpret_cast<float*>(sm.w[0]);            // [128 channels][TLD]
    float* ztv = reinterpret_cast<float*>(sm.red);              // [128] (z^T Phi)[f]
    static_assert(sizeof(sm.w) + sizeof(sm.a) >= 128 * TLD * sizeof(float), "transpose tile");
    static_assert(sizeof(sm.red) >= 128 * sizeof(float), "z^T Phi row");
    const int cch = 32 * (warp & 3) + lane;  // TMEM lane = value channel
#pragma unroll 1
    for (int c0 = 64 * part; c0 < 64 * part + 64; c0 += 32) {
      float d[32];
      tc::tmem_ld32(lane_addr + FT_COL_S + 128 * hp + c0, reinterpret_cast<uint32_t*>(d));
      tc::wait_ld();
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(tile + cch * TLD + c0 + i) = make_float4(d[i], d[i + 1], d[i + 2], d[i + 3]);
    }
    if (tid < HALF) {
      const int f = tid;
      ztv[f] = zf[G + f];
    }
    __syncthreads();
    FT_DRAIN(2);
    // all 16 row pieces of the thread loaded before any store (a load after a store to S
    // cannot be hoisted by the compiler: one L2 round trip per piece, ~10k cycles per half)
    constexpr int NPC = 128 * 32 / FT_THREADS;
    float4 old[NPC];
#pragma unroll
    for (int k = 0; k < NPC; ++k) {
      const int idx = tid + k * FT_THREADS, r = idx >> 5, f4 = (idx & 31) * 4;
      old[k] = __ldcg(reinterpret_cast<const float4*>(S + (size_t)r * RANK + h * HALF + f4));
    }
#pragma unroll
    for (int k = 0; k < NPC; ++k) {
      const int idx = tid + k * FT_THREADS, r = idx >> 5, f4 = (idx & 31) * 4;
      const float4 t4 = *reinterpret_cast<const float4*>(tile + r * TLD + f4);
      const float4 z4 = *reinterpret_cast<const float4*>(ztv + f4);
      float4 o = old[k];
      o.x += t4.x + z4.x;
      o.y += t4.y + z4.y;
      o.z += t4.z + z4.z;
      o.w += t4.w + z4.w;
      *reinterpret_cast<float4*>(S + (size_t)r * RANK + h * HALF + f4) = o;
    }
  }
  FT_DRAIN(3);
  }
  tc::fence_before_sync();
  __syncthreads();
  FT_PHASE(3);
  if (warp == 0) tc::tmem_dealloc(tb, FT_TMEM2);
}


#ifdef KVLC_TRACE
}  // namespace
int kvlc_qtok_copy(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_qtok, bytes < sizeof(g_qtok) ? bytes : sizeof(g_qtok)) == cudaSuccess ? 0 : 2;
}
int kvlc_qtrace_copy(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_qtrace, bytes < sizeof(g_qtrace) ? bytes : sizeof(g_qtrace)) == cudaSuccess ? 0 : 2;
}
int kvlc_ftrace_copy(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_ftrace, bytes < sizeof(g_ftrace) ? bytes : sizeof(g_ftrace)) == cudaSuccess ? 0 : 2;
}
namespace {
#endif
// The tensor-core flush (quant_kernel -> flush_tc_kernel -> reduce_state) of the chunks
// seq.nflush[b] per sequence; `a` carries the source (prefill tokens or the ring).  The
// workspace is kvlc_prefill_workspace(c, n_tok) bytes.
int launch_tc_flush(const kvlc_cache* c, const kvlc_adapter* ad, FlushArgs a, const SeqInfo& seq, int max_nf,
                    int64_t n_tok, void* ws, size_t ws_bytes, cudaStream_t s) {
  int rc = 0;
  const int units = c->B * c->Hkv;
  static int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int ws_splits = (int)std::max<int64_t>(1, (n_tok / KVLC_G + 3) / 4);  // kvlc_prefill_workspace bound
  // enough CTAs to fill whole waves (2 per unit-split: the feature halves), and at most 32
  // chunks accumulated per TMEM partial: 63-chunk partials (an 8k sequence in a 128-unit
  // batch) drifted to 1.3e-5 relative (T3 is 1e-5), 32-chunk ones measure 8e-6, 16-chunk
  // ones 6e-6 but cost config 5 ~40 us in extra CTAs (tools/s_error_c2.py)
#ifndef KVLC_TC_MAXCPC
#define KVLC_TC_MAXCPC 32
#endif
  static const int both_env = [] {  // KVLC_FT_BOTH: 0 off, 1 ring flushes (default), 2 always
    const char* e = getenv("KVLC_FT_BOTH");
    return e ? atoi(e) : 1;
  }();
  const int per = both_env == 2 ? 1 : 2;  // state CTAs per (unit, chunk range)
  const int base = std::max({1, std::min(max_nf, sms / (per * units)), (max_nf + KVLC_TC_MAXCPC - 1) / KVLC_TC_MAXCPC});
  const int waves = (per * units * base + sms - 1) / sms;  // one CTA per SM: fill the last wave
  const int splits = std::min({ws_splits, std::max(1, max_nf), std::max(base, waves * sms / (per * units))});
  const int cpc = (max_nf + splits - 1) / splits;
  // one CTA per (unit, feature half): it adds its S / P straight into the cache (the halves
  // write disjoint columns), no partials, memset or reduction (decode-time ring flushes)
  const bool direct = splits == 1;
  Arena ar(ws, ws_bytes);
  float* s_part = ar.take<float>((size_t)units * splits * (D * RANK + RANK));
  uint8_t* wtiles = ar.take<uint8_t>((size_t)c->Hkv * 2 * 2 * FT_TILE);
  const int slot_stride = (int)std::max<int64_t>(1, n_tok / KVLC_G);
  uint8_t* aimg = ar.take<uint8_t>((size_t)units * slot_stride * 2 * FT_TILE);
  uint8_t* cimg = ar.take<uint8_t>((size_t)units * slot_stride * FT_TILE);
  float2* vsz = ar.take<float2>((size_t)units * slot_stride * G);
  KVLC_REQUIRE(s_part && wtiles && aimg && cimg && vsz, "flush workspace too small (%zu bytes)", ws_bytes);
  float* p_part = s_part + (size_t)units * splits * D * RANK;
  if (!direct) KVLC_CUDA(cudaMemsetAsync(s_part, 0, (size_t)units * splits * (D * RANK + RANK) * sizeof(float), s));
  a.wtiles = wtiles;
  a.prep_n = 16 * c->Hkv * 2;
  a.c = *c;
  a.ad = *ad;
  a.use_adapter = 1;
  a.cpc = cpc;
  a.s_out = direct ? nullptr : s_part;
  a.p_out = direct ? nullptr : p_part;
  a.splits = splits;
  a.aimg = aimg;
  a.cimg = cimg;
  a.vsz = vsz;
  a.slot_stride = slot_stride;
  // decode-time ring flushes (one chunk per unit, grid below one wave): the value tokens of a
  // chunk over 4 more CTAs, keys in the first (latency, not throughput, sets that step)
  static const int vsplit_env = [] {
    const char* e = getenv("KVLC_VSPLIT");
    return e ? atoi(e) : -1;
  }();
  // value CTAs per chunk: enough that K1 (the key CTA) sets the time, few enough that key and
  // value CTAs fit one wave of quant_kernel's 3 CTAs per SM
  int vs = 4;
  while (vs > 1 && (long long)units * (1 + vs) > 3LL * sms) vs >>= 1;
  if (vsplit_env >= 0) vs = vsplit_env;
  a.vsplit = (a.ring && max_nf == 1 && vs > 0) ? vs : 0;
  KVLC_CUDA(cudaFuncSetAttribute(quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(QkSmem)));
  quant_kernel<<<dim3(max_nf, units, a.vsplit ? 1 + a.vsplit : 1), FT_THREADS, sizeof(QkSmem), s>>>(a, seq);
  if ((rc = check_launch("quant"))) return rc;
  KVLC_CUDA(cudaFuncSetAttribute(flush_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FtSmem)));
  // one chunk per unit (decode-time ring flush): both feature halves in one CTA
  a.both = (both_env == 2 || (a.ring && max_nf == 1 && splits == 1 && both_env)) ? 1 : 0;
  flush_tc_kernel<<<dim3(splits, units, a.both ? 1 : 2), FT_THREADS, sizeof(FtSmem), s>>>(a, seq, wtiles);
  if ((rc = check_launch("flush_tc"))) return rc;
  if (direct) return KVLC_OK;
  reduce_state_kernel<<<dim3(32, units), 256, 0, s>>>(*c, s_part, p_part, splits);
  return check_launch("reduce_state");
}

int check_cache(const kvlc_cache* c) {
  KVLC_REQUIRE(c != nullptr, "null cache descriptor");
  KVLC_REQUIRE(c->B >= 1 && c->Hkv >= 1 && c->Hq >= c->Hkv && c->Hq % c->Hkv == 0 &&
                   c->Hq / c->Hkv <= 8,
               "bad cache dims B=%d Hkv=%d Hq=%d (GQA group must divide and be <= 8)", c->B,
               c->Hkv, c->Hq);
  KVLC_REQUIRE(c->kcodes && c->vcodes && c->kscale && c->kzero && c->vscale && c->vzero &&
                   c->kres && c->vres && c->S && c->P && c->n_chunks && c->res_start && c->res_len,
               "cache descriptor has null buffers");
  return KVLC_OK;
}

bool adapter_on(const kvlc_adapter* ad) {
  return ad != nullptr && ad->enabled && ad->w1k && ad->w2k && ad->w1q && ad->w2q;
}

}  // namespace
}  // namespace kvlc

using namespace kvlc;

extern "C" {

size_t kvlc_prefill_workspace(const kvlc_cache* c, int64_t n_tok) {
  if (!c) return 0;
  int64_t nf = n_tok / KVLC_G;
  int units = c->B * c->Hkv;
  int splits = (int)((nf + 3) / 4);
  if (splits < 1) splits = 1;
  // S / P partials (the tensor-core path uses fewer splits) + the W hi / lo tiles +
  // the quant_kernel -> state-kernel operands (A_phi hi / lo 64 KB, fp16 codes 32 KB and the
  // value (scale, zero) 1 KB per chunk)
  const size_t nslot = (size_t)units * std::max<int64_t>(nf, 1);
  return align_up((size_t)units * splits * (D * RANK + RANK) * sizeof(float)) +
         align_up((size_t)c->Hkv * 2 * 2 * FT_TILE) + align_up(nslot * 2 * FT_TILE) + align_up(nslot * FT_TILE) +
         align_up(nslot * G * sizeof(float2));
}

int kvlc_prefill(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* k, const uint16_t* v,
                 int64_t n_tok, const int32_t* lens_host, int32_t keep_window, void* ws, size_t ws_bytes,
                 void* stream) {
  KVLC_NEED_DEVICE();
  int rc = check_cache(c);
  if (rc) return rc;
  KVLC_REQUIRE(c->B <= MAX_B, "batch %d exceeds the supported %d sequences", c->B, MAX_B);
  cudaStream_t s = as_stream(stream);
  const int units = c->B * c->Hkv;
  kvlc::note_cache_write(c);  // codes and chunk counts change: the next decode waits fully
  static thread_local SeqInfo seq;
  memset(&seq, 0, sizeof(seq));
  int max_nf = 0;
  for (int b = 0; b < c->B; ++b) {
    KVLC_REQUIRE(lens_host[b] >= 0 && lens_host[b] <= n_tok, "sequence length %d out of range", lens_host[b]);
    int nf = keep_window ? (lens_host[b] >= KVLC_R ? (lens_host[b] - KVLC_R) / KVLC_G : 0)
                         : lens_host[b] / KVLC_G;
    KVLC_REQUIRE(nf <= c->max_chunks, "prefill of %d tokens exceeds capacity of %d chunks",
                 lens_host[b], c->max_chunks);
    seq.nflush[b] = nf;
    seq.len[b] = lens_host[b];
    if (nf > max_nf) max_nf = nf;
  }
  const bool use_ad = adapter_on(ad);
  if (max_nf > 0 && use_ad) {
    FlushArgs a{};
    a.ksrc = k;
    a.vsrc = v;
    a.k_unit = n_tok * D;
    a.k_t = D;
    a.k_c = 1;
    a.v_unit = n_tok * D;
    a.v_t = D;
    a.v_c = 1;
    a.ring = 0;
    if ((rc = launch_tc_flush(c, ad, a, seq, max_nf, n_tok, ws, ws_bytes, s))) return rc;
  } else if (max_nf > 0) {
    // cpc chunks per CTA: enough CTAs to cover the SMs
    const int cpc = 4;
    const int splits = (max_nf + cpc - 1) / cpc;
    FlushArgs a{};
    a.c = *c;
    a.use_adapter = 0;
    a.ksrc = k;
    a.vsrc = v;
    a.k_unit = n_tok * D;
    a.k_t = D;
    a.k_c = 1;
    a.v_unit = n_tok * D;
    a.v_t = D;
    a.v_c = 1;
    a.ring = 0;
    a.cpc = cpc;
    a.splits = splits;
    KVLC_CUDA(cudaFuncSetAttribute(flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FLUSH_SMEM));
    flush_kernel<<<dim3(splits, units), FLUSH_THREADS, FLUSH_SMEM, s>>>(a, seq);
    if ((rc = check_launch("flush"))) return rc;
  }
  load_residual_kernel<<<dim3(64, units), 256, 0, s>>>(*c, k, v, n_tok, seq);
  set_lengths_kernel<<<1, 256, 0, s>>>(*c, seq);
  return check_launch("prefill");
}

size_t kvlc_append_workspace(const kvlc_cache* c) { return kvlc_prefill_workspace(c, KVLC_G); }

int kvlc_append(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* k_t, const uint16_t* v_t,
                const int32_t* active_host, const int32_t* flush_host, void* ws, size_t ws_bytes,
                void* stream) {
  KVLC_NEED_DEVICE();
  int rc = check_cache(c);
  if (rc) return rc;
  KVLC_REQUIRE(c->B <= MAX_B, "batch %d exceeds the supported %d sequences", c->B, MAX_B);
  cudaStream_t s = as_stream(stream);
  static thread_local SeqInfo seq;
  memset(seq.active, 0, sizeof(seq.active));
  memset(seq.flush, 0, sizeof(seq.flush));
  memset(seq.nflush, 0, sizeof(seq.nflush));
  bool any_flush = false;
  for (int b = 0; b < c->B; ++b) {
    if (!active_host || active_host[b]) seq.active[b >> 5] |= 1u << (b & 31);
    if (flush_host && flush_host[b]) {
      seq.flush[b >> 5] |= 1u << (b & 31);
      seq.nflush[b] = 1;
      any_flush = true;
    }
  }
  // a flush writes codes / chunk counts, which the next decode reads before its
  // griddepcontrol.wait: that decode must not overlap (a plain append only moves the
  // residual ring, read after the wait)
  if (any_flush) kvlc::note_cache_write(c);
  const int units = c->B * c->Hkv;
  append_kernel<<<units, D, 0, s>>>(*c, k_t, v_t, seq);
  if ((rc = check_launch("append"))) return rc;
  if (any_flush && adapter_on(ad) && ws && ws_bytes >= kvlc_append_workspace(c)) {
    // tensor-core flush of the due sequences' oldest G ring slots (quant_kernel in ring mode)
    FlushArgs a{};
    a.ksrc = c->kres;
    a.vsrc = c->vres;
    a.k_unit = (int64_t)SLOTS * D;
    a.k_t = D;
    a.k_c = 1;
    a.v_unit = (int64_t)D * SLOTS;
    a.v_t = 1;
    a.v_c = SLOTS;
    a.ring = 1;
    a.finalize = 1;  // the ring counters move in flush_tc_kernel's first CTA
    if ((rc = launch_tc_flush(c, ad, a, seq, 1, KVLC_G, ws, ws_bytes, s))) return rc;
    return KVLC_OK;
  } else if (any_flush) {
    const bool use_ad = adapter_on(ad);
    FlushArgs a{};
    a.c = *c;
    if (use_ad) a.ad = *ad;
    a.use_adapter = use_ad ? 1 : 0;
    a.ksrc = c->kres;
    a.vsrc = c->vres;
    a.k_unit = (int64_t)SLOTS * D;
    a.k_t = D;
    a.k_c = 1;
    a.v_unit = (int64_t)D * SLOTS;
    a.v_t = 1;
    a.v_c = SLOTS;
    a.ring = 1;
    a.cpc = 1;
    a.splits = 1;
    KVLC_CUDA(cudaFuncSetAttribute(flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FLUSH_SMEM));
    flush_kernel<<<dim3(1, units), FLUSH_THREADS, FLUSH_SMEM, s>>>(a, seq);
    if ((rc = check_launch("flush"))) return rc;
  }
  append_finalize_kernel<<<1, 256, 0, s>>>(*c, seq);
  return check_launch("append_finalize");
}

size_t kvlc_unit_image_bytes(int32_t n_chunks, int32_t res_len, int32_t rank) {
  if (n_chunks < 0 || res_len < 0 || res_len > SLOTS || !(rank == 0 || rank == RANK)) return 0;
  return ImageLayout(n_chunks, res_len, rank).end;
}

int kvlc_serialize_unit(const kvlc_cache* c, int32_t unit, int32_t n_chunks, int32_t res_start, int32_t res_len,
                        int32_t rank, uint8_t* image, void* stream) {
  KVLC_NEED_DEVICE();
  int rc = check_cache(c);
  if (rc) return rc;
  KVLC_REQUIRE(unit >= 0 && unit < c->B * c->Hkv, "unit %d out of range", unit);
  KVLC_REQUIRE(n_chunks >= 0 && n_chunks <= c->max_chunks, "%d chunks exceeds capacity of %d chunks", n_chunks,
               c->max_chunks);
  KVLC_REQUIRE(res_len >= 0 && res_len <= SLOTS && res_start >= 0 && res_start < SLOTS, "residual range (%d, %d)",
               res_start, res_len);
  KVLC_REQUIRE(rank == 0 || rank == RANK, "cache state rank %d (serving cache holds %d)", rank, RANK);
  serialize_unit_kernel<<<n_chunks + 1 + (rank ? 32 : 0), 256, 0, as_stream(stream)>>>(*c, unit, n_chunks, res_start,
                                                                                          res_len, rank, image);
  return check_launch("serialize_unit");
}

int kvlc_deserialize_unit(const kvlc_cache* c, int32_t unit, const uint8_t* image, int32_t n_chunks,
                          int32_t res_len, int32_t rank, void* stream) {
  KVLC_NEED_DEVICE();
  int rc = check_cache(c);
  if (rc) return rc;
  kvlc::note_cache_write(c);  // no PDL overlap for the next decode of this cache
  KVLC_REQUIRE(unit >= 0 && unit < c->B * c->Hkv, "unit %d out of range", unit);
  KVLC_REQUIRE(n_chunks >= 0 && n_chunks <= c->max_chunks, "cache of %d chunks exceeds capacity of %d chunks",
               n_chunks, c->max_chunks);
  KVLC_REQUIRE(res_len >= 0 && res_len <= SLOTS, "residual length %d exceeds the ring (%d)", res_len, SLOTS);
  KVLC_REQUIRE(rank == 0 || rank == RANK, "cache state rank %d (serving cache holds %d)", rank, RANK);
  deserialize_unit_kernel<<<n_chunks + 1 + 32, 256, 0, as_stream(stream)>>>(*c, unit, n_chunks, res_len, rank, image);
  return check_launch("deserialize_unit");
}

int kvlc_export_chunk(const kvlc_cache* c, int32_t unit, int32_t chunk, uint32_t* kwords,
                      uint32_t* vwords, uint16_t* kscale, uint16_t* kzero, uint16_t* vscale,
                      uint16_t* vzero, void* stream) {
  KVLC_NEED_DEVICE();
  int rc = check_cache(c);
  if (rc) return rc;
  KVLC_REQUIRE(unit >= 0 && unit < c->B * c->Hkv && chunk >= 0 && chunk < c->max_chunks,
               "chunk (%d, %d) out of range", unit, chunk);
  export_chunk_kernel<<<1, 256, 0, as_stream(stream)>>>(*c, unit, chunk, kwords, vwords, kscale, kzero, vscale, vzero);
  return check_launch("export_chunk");
}

}  // extern "C"
