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
#include "kvlc_common.cuh"

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
  return (words[((w * 32) + 4 * g + t0) * 8 + kt] >> (8 * q + 2 * j)) & 3u;
}

__device__ __forceinline__ uint32_t v_code(const uint32_t* words, int t, int c) {
  const int w = t >> 5, u = t & 31, t0 = u >> 3, hi = (u >> 2) & 1, mt = (u >> 1) & 1, lo = u & 1;
  const int q = lo + 2 * hi, g = c & 7, r = (c >> 3) & 1, mv = c >> 4, p = mv >> 1, j = 2 * (mv & 1) + r;
  return (words[((w * 32) + 4 * g + t0) * 8 + 4 * mt + p] >> (8 * q + 2 * j)) & 3u;
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
    for (int wi = tid; wi < 1024; wi += FLUSH_THREADS) c.kcodes[cb * 1024 + wi] = pack_k_word(codes_s, wi);
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
          x[e] = (lane & k) ? (o - x[e]) : (x[e] + o);
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
    for (int wi = tid; wi < 1024; wi += FLUSH_THREADS) c.vcodes[cb * 1024 + wi] = pack_v_word(codes_s, wi);
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

__global__ void append_finalize_kernel(kvlc_cache c, const SeqInfo seq) {
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
  return align_up((size_t)units * splits * (D * RANK + RANK) * sizeof(float));
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
  // cpc chunks per CTA: enough CTAs to cover the SMs, few enough partials
  const int cpc = 4;
  const int splits = max_nf > 0 ? (max_nf + cpc - 1) / cpc : 1;
  const bool use_ad = adapter_on(ad);
  if (max_nf > 0) {
    float *s_part = nullptr, *p_part = nullptr;
    if (use_ad) {
      Arena ar(ws, ws_bytes);
      s_part = ar.take<float>((size_t)units * splits * (D * RANK + RANK));
      KVLC_REQUIRE(s_part, "prefill workspace too small (%zu bytes)", ws_bytes);
      p_part = s_part + (size_t)units * splits * D * RANK;
      KVLC_CUDA(cudaMemsetAsync(s_part, 0, (size_t)units * splits * (D * RANK + RANK) * sizeof(float), s));
    }
    FlushArgs a{};
    a.c = *c;
    if (use_ad) a.ad = *ad;
    a.use_adapter = use_ad ? 1 : 0;
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
    a.s_out = s_part;
    a.p_out = p_part;
    a.splits = splits;
    KVLC_CUDA(cudaFuncSetAttribute(flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FLUSH_SMEM));
    flush_kernel<<<dim3(splits, units), FLUSH_THREADS, FLUSH_SMEM, s>>>(a, seq);
    if ((rc = check_launch("flush"))) return rc;
    if (use_ad) {
      reduce_state_kernel<<<dim3(32, units), 256, 0, s>>>(*c, s_part, p_part, splits);
      if ((rc = check_launch("reduce_state"))) return rc;
    }
  }
  load_residual_kernel<<<dim3(64, units), 256, 0, s>>>(*c, k, v, n_tok, seq);
  set_lengths_kernel<<<1, 256, 0, s>>>(*c, seq);
  return check_launch("prefill");
}

int kvlc_append(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* k_t, const uint16_t* v_t,
                const int32_t* active_host, const int32_t* flush_host, void* ws, size_t ws_bytes,
                void* stream) {
  (void)ws;
  (void)ws_bytes;
  KVLC_NEED_DEVICE();
  int rc = check_cache(c);
  if (rc) return rc;
  KVLC_REQUIRE(c->B <= MAX_B, "batch %d exceeds the supported %d sequences", c->B, MAX_B);
  cudaStream_t s = as_stream(stream);
  static thread_local SeqInfo seq;
  memset(seq.active, 0, sizeof(seq.active));
  memset(seq.flush, 0, sizeof(seq.flush));
  bool any_flush = false;
  for (int b = 0; b < c->B; ++b) {
    if (!active_host || active_host[b]) seq.active[b >> 5] |= 1u << (b & 31);
    if (flush_host && flush_host[b]) {
      seq.flush[b >> 5] |= 1u << (b & 31);
      any_flush = true;
    }
  }
  const int units = c->B * c->Hkv;
  append_kernel<<<units, D, 0, s>>>(*c, k_t, v_t, seq);
  if ((rc = check_launch("append"))) return rc;
  if (any_flush) {
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
