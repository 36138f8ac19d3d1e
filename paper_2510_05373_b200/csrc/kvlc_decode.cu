// Fused KVLinC decode for the batched serving cache (d = G = 128, 2-bit).
//
// Reference: decode_step_blocked (attention.py:197-276) = Algorithm 1
// (PAPER.md:172-199): per-block fp32 scores / max / exp / partial numerators
// over the quantized history, one extra full-precision block for the
// residual window, the phi_q(q)·S / phi_q(q)·P correction folded with the
// e^{-M}-consistent rule (_reduce_blocks, attention.py:158-194), the inverse
// Hadamard rotation of the quantized numerator and the final divide.
//
// Kernels (one decode step = 3 launches, PDL-chained):
//   phi_kernel      phi_q(q) per q-head and C_d = P . phi      (attention.py:224-228)
//   split_kernel    per CTA task, warp-specialised by blockIdx:
//                   * quantized split: chunks of one (b, kv-head) unit, GQA
//                     heads batched on the MMA N dimension, 2-bit codes turned
//                     into fp16 MMA operands by one LOP3 each (exact subnormal
//                     values c * 4^j * 2^-24), scales folded into q / p
//                     (hi+lo fp16 split when the group has <= 4 heads)
//                   * residual half: bf16 ring window, masked
//                   * correction rows: C_n = S phi for 32 rows of S
//   combine_kernel  LSE merge of the split records + correction, warp FWHT
//                   (H^T = H), divide, bf16 out.
//
// Online-softmax state is kept in log2 units (logit * log2 e); the sign of the
// global max, which selects the correction branch, is unit independent.
#include "kvlc_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace kvlc {
namespace {

constexpr int D = KVLC_D;
constexpr int G = KVLC_G;
constexpr int SLOTS = KVLC_SLOTS;
constexpr int RANK = KVLC_RANK;
constexpr int HALF = RANK / 2;
constexpr int WARPS = 4;
constexpr int THREADS = WARPS * 32;
constexpr int REC = 4 + D;  // record: m (log2 units), l, pad, pad, y[D] (16-byte aligned y)
constexpr int PREC = 4 + 2 * D;  // device-partial record: m, l, pad, pad, y_rot[D], y_raw[D]
constexpr float LOG2E = 1.4426950408889634f;
constexpr float C0 = 0.12751743074173226f;  // log2(e) / sqrt(128)
constexpr int CORR_ROWS = 32;               // S rows per correction CTA
constexpr int CORR_CTAS = D / CORR_ROWS;

__device__ __forceinline__ float bf2f(uint16_t x) { return __uint_as_float((uint32_t)x << 16); }

__device__ __forceinline__ void mma_f16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                        uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

__device__ __forceinline__ uint4 ldg4(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ uint2 ldg2(const void* p) {
  return __ldg(reinterpret_cast<const uint2*>(p));
}
__device__ __forceinline__ uint32_t w4(const uint4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// byte b of x into byte 0 and byte b of y into byte 2 (bytes 1, 3 are masked off later)
__device__ __forceinline__ uint32_t pick(uint32_t x, uint32_t y, int b) {
  return __byte_perm(x, y, (uint32_t)(b | (b << 4) | ((4 + b) << 8) | ((4 + b) << 12)));
}
// half2 of fp16 subnormals (c_lo * 4^j * 2^-24, c_hi * 4^j * 2^-24)
__device__ __forceinline__ uint32_t code_h2(uint32_t x, int j) { return x & (0x00030003u << (2 * j)); }

// 2^24 * 4^-j
__device__ __forceinline__ constexpr float code_unscale(int j) {
  return j == 0 ? 16777216.f : (j == 1 ? 4194304.f : (j == 2 ? 1048576.f : 262144.f));
}

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n"); }

struct DecArgs {
  kvlc_cache c;
  const uint16_t* q;      // [B][Hq][D] bf16
  const float* phi;       // [B][Hq][RANK]
  float* corr;            // [B][Hq][1 + D]  (C_d, C_n)
  float* rec;             // [U][nrec][NG][REC]
  int nsq;                // quantized split CTAs per unit
  int cpw;                // chunks per warp
  int chunk_lo, chunk_hi; // global chunk window (split-KV across devices)
  int tail;               // include residual window + correction rows
  int corr_on;            // adapter active
  int nrec;               // records per unit = nsq + 2*tail
};

// ---------------------------------------------------------------- phi_q ----
template <int NG>
__global__ void __launch_bounds__(256) phi_kernel(kvlc_cache c, const float* __restrict__ w1q,
                                                  const float* __restrict__ w2q,
                                                  const uint16_t* __restrict__ q,
                                                  float* __restrict__ phi, float* __restrict__ corr) {
  griddep_launch();
  __shared__ float qs[NG][D];
  __shared__ float red[8][NG];
  __shared__ float stat[2][NG];
  const int unit = blockIdx.x, b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int f = threadIdx.x, warp = f >> 5, lane = f & 31, half = f >> 7;
  const size_t qbase = ((size_t)b * c.Hq + (size_t)kvh * NG) * D;
  for (int i = f; i < NG * D; i += 256) qs[i / D][i % D] = bf2f(q[qbase + i]);
  __syncthreads();
  const float* W = (half ? w2q : w1q) + (size_t)kvh * D * HALF + (f & (HALF - 1));
  float acc[NG];
#pragma unroll
  for (int i = 0; i < NG; ++i) acc[i] = 0.f;
  for (int ch = 0; ch < D; ++ch) {
    float w = __ldg(W + ch * HALF);
#pragma unroll
    for (int i = 0; i < NG; ++i) acc[i] = fmaf(qs[i][ch], w, acc[i]);
  }
  // max-shifted softmax within each half (linalg.py:38-47)
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    float m = warp_max(acc[i]);
    if (lane == 0) red[warp][i] = m;
  }
  __syncthreads();
  if (f < 2 * NG) {
    int h = f / NG, i = f % NG;
    float m = red[4 * h][i];
    for (int w = 1; w < 4; ++w) m = fmaxf(m, red[4 * h + w][i]);
    stat[h][i] = m;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NG; ++i) acc[i] = expf(acc[i] - stat[half][i]);
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    float s = warp_sum(acc[i]);
    if (lane == 0) red[warp][i] = s;
  }
  __syncthreads();
  if (f < 2 * NG) {
    int h = f / NG, i = f % NG;
    float s = 0.f;
    for (int w = 0; w < 4; ++w) s += red[4 * h + w][i];
    stat[h][i] = s;
  }
  __syncthreads();
  const float pf = c.P[(size_t)unit * RANK + f];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    float ph = acc[i] / stat[half][i];
    phi[(qbase / D + i) * RANK + f] = ph;
    acc[i] = pf * ph;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    float s = warp_sum(acc[i]);
    if (lane == 0) red[warp][i] = s;
  }
  __syncthreads();
  if (f < NG) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red[w][f];
    corr[(qbase / D + f) * (1 + D)] = s;  // C_d
  }
}

// ------------------------------------------------------ per-warp state ----
// Heads handled per thread in the C layout: HILO -> head t; else heads 2t, 2t+1.
template <int NG>
struct WarpState {
  static constexpr bool HILO = NG <= 4;
  static constexpr int NH = HILO ? 1 : 2;
  float m[NH], l[NH], z[NH];
  float acc[8][4];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int e = 0; e < NH; ++e) {
      m[e] = -INFINITY;
      l[e] = 0.f;
      z[e] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  }
};

// One quantized chunk (128 tokens) for one warp.
// EXTRA (groups of > 4 heads only): bit 0 adds a low-part pass to Q K^T,
// bit 1 adds a low-part pass to P V (hi + lo fp16 operands, two MMAs).
template <int NG, int EXTRA>
__device__ __forceinline__ void quant_chunk(const kvlc_cache& c, size_t cb, const uint32_t (&qh)[8][2],
                                            WarpState<NG>& st, int lane) {
  constexpr bool HILO = NG <= 4;
  constexpr bool QK_LO = !HILO && (EXTRA & 1);
  constexpr bool PV_LO = !HILO && (EXTRA & 2);
  const int g = lane >> 2, t = lane & 3;
  // ---- loads: K words (word row g, channels 16kt+4t..+3), K meta, V words (row g, slots 16i+4t..) ----
  uint4 kw[8], vw[8];
  uint2 ks[8], kz[8];
  const uint32_t* kc = c.kcodes + (cb * 8 + g) * 128 + 4 * t;
  const uint32_t* vc = c.vcodes + (cb * 8 + g) * 128 + 4 * t;
#pragma unroll
  for (int i = 0; i < 8; ++i) kw[i] = ldg4(kc + 16 * i);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ks[i] = ldg2(c.kscale + cb * D + 16 * i + 4 * t);
    kz[i] = ldg2(c.kzero + cb * D + 16 * i + 4 * t);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) vw[i] = ldg4(vc + 16 * i);
  const uint4 vs0 = ldg4(c.vscale + cb * G + 16 * g), vs1 = ldg4(c.vscale + cb * G + 16 * g + 8);
  const uint4 vz0 = ldg4(c.vzero + cb * G + 16 * g), vz1 = ldg4(c.vzero + cb * G + 16 * g + 8);

  // ---- B operand for QK: q' = q * s_k (hi / lo fp16), and zt = q . z_k ----
  uint32_t bq[8][2];
  uint32_t bql[QK_LO ? 8 : 1][2];
  float zp = 0.f;
  const __half2 lo_mask = (HILO && (g & 1)) ? u2h(0xffffffffu) : u2h(0u);
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      __half2 qv = u2h(qh[kt][e]);
      __half2 sv = u2h(e ? ks[kt].y : ks[kt].x);
      __half2 hi = __hmul2(qv, sv);
      if (HILO) {
        // odd columns carry the low part q*s - hi (exact FMA residual)
        uint32_t neg = (h2u(hi) ^ 0x80008000u) & h2u(lo_mask);
        __half2 r = __hfma2(qv, sv, u2h(neg));
        bq[kt][e] = h2u(r);
      } else {
        bq[kt][e] = h2u(hi);
        if (QK_LO) bql[kt][e] = h2u(__hfma2(qv, sv, __hneg2(hi)));
      }
      float2 qf = __half22float2(qv);
      float2 zf = __half22float2(u2h(e ? kz[kt].y : kz[kt].x));
      zp = fmaf(qf.x, zf.x, zp);
      zp = fmaf(qf.y, zf.y, zp);
    }
  }
  zp += __shfl_xor_sync(0xffffffffu, zp, 1);
  zp += __shfl_xor_sync(0xffffffffu, zp, 2);
  float zt[WarpState<NG>::NH];
  if (HILO) {
    zt[0] = __shfl_sync(0xffffffffu, zp, 8 * t) * C0;
  } else {
    zt[0] = __shfl_sync(0xffffffffu, zp, 8 * t) * C0;
    zt[1] = __shfl_sync(0xffffffffu, zp, 8 * t + 4) * C0;
  }

  // ---- QK^T: 8 token tiles x 8 channel tiles ----
  float cq[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cq[i][j] = 0.f;
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) {
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      uint32_t x0 = pick(kw[kt].x, kw[kt].y, bb), x1 = pick(kw[kt].z, kw[kt].w, bb);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int mt = 2 * bb + h;
        mma_f16(cq[mt], code_h2(x0, 2 * h), code_h2(x0, 2 * h + 1), code_h2(x1, 2 * h),
                code_h2(x1, 2 * h + 1), bq[kt][0], bq[kt][1]);
        if (QK_LO)
          mma_f16(cq[mt], code_h2(x0, 2 * h), code_h2(x0, 2 * h + 1), code_h2(x1, 2 * h),
                  code_h2(x1, 2 * h + 1), bql[QK_LO ? kt : 0][0], bql[QK_LO ? kt : 0][1]);
      }
    }
  }

  // ---- online softmax over this chunk (tokens 16g + 2mt + r) ----
  constexpr int NH = WarpState<NG>::NH;
  float cmax[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) cmax[e] = -INFINITY;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float F = code_unscale(2 * (mt & 1) + r) * C0;
      if (HILO) {
        float v = fmaf(cq[mt][2 * r] + cq[mt][2 * r + 1], F, zt[0]);
        cq[mt][2 * r] = v;
        cmax[0] = fmaxf(cmax[0], v);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float v = fmaf(cq[mt][2 * r + e], F, zt[e]);
          cq[mt][2 * r + e] = v;
          cmax[e] = fmaxf(cmax[e], v);
        }
      }
    }
  }
  float sc[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) {
    float m = cmax[e];
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
    float mn = fmaxf(st.m[e], m);
    sc[e] = exp2f(st.m[e] - mn);
    st.m[e] = mn;
    st.l[e] *= sc[e];
    st.z[e] *= sc[e];
  }
#pragma unroll
  for (int mv = 0; mv < 8; ++mv) {
    if (HILO) {
#pragma unroll
      for (int j = 0; j < 4; ++j) st.acc[mv][j] *= sc[0];
    } else {
      st.acc[mv][0] *= sc[0];
      st.acc[mv][2] *= sc[0];
      st.acc[mv][1] *= sc[1];
      st.acc[mv][3] *= sc[1];
    }
  }
  // p, l, z and the PV B operand p' = p * s_v (hi/lo or two heads), transposed by movmatrix
  uint32_t bp[8][2];
  uint32_t bpl[PV_LO ? 8 : 1][2];
  const uint32_t vsw[8] = {vs0.x, vs0.y, vs0.z, vs0.w, vs1.x, vs1.y, vs1.z, vs1.w};
  const uint32_t vzw[8] = {vz0.x, vz0.y, vz0.z, vz0.w, vz1.x, vz1.y, vz1.z, vz1.w};
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const float2 s2 = __half22float2(u2h(vsw[mt]));  // tokens 2mt, 2mt+1
    const float2 z2 = __half22float2(u2h(vzw[mt]));
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float sv = r ? s2.y : s2.x, zv = r ? z2.y : z2.x;
      uint32_t packed;
      if (HILO) {
        float p = exp2f(cq[mt][2 * r] - st.m[0]);
        st.l[0] += p;
        st.z[0] = fmaf(p, zv, st.z[0]);
        float pv = p * sv;
        __half hi = __float2half_rn(pv);
        __half lo = __float2half_rn(pv - __half2float(hi));
        packed = h2u(__halves2half2(hi, lo));
      } else {
        float p0 = exp2f(cq[mt][2 * r] - st.m[0]);
        float p1 = exp2f(cq[mt][2 * r + 1] - st.m[1]);
        st.l[0] += p0;
        st.l[1] += p1;
        st.z[0] = fmaf(p0, zv, st.z[0]);
        st.z[1] = fmaf(p1, zv, st.z[1]);
        const float a0 = p0 * sv, a1 = p1 * sv;
        const __half2 hh = __floats2half2_rn(a0, a1);
        packed = h2u(hh);
        if (PV_LO) {
          const float2 hf = __half22float2(hh);
          bpl[PV_LO ? mt : 0][r] = movm_t(h2u(__floats2half2_rn(a0 - hf.x, a1 - hf.y)));
        }
      }
      bp[mt][r] = movm_t(packed);
    }
  }

  // ---- P V: 8 channel tiles x 8 token tiles ----
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const int i0 = mt >> 1, ln = 2 * (mt & 1);
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      uint32_t x0 = pick(w4(vw[i0], ln), w4(vw[4 + i0], ln), bb);
      uint32_t x1 = pick(w4(vw[i0], ln + 1), w4(vw[4 + i0], ln + 1), bb);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int mv = 2 * bb + h;
        mma_f16(st.acc[mv], code_h2(x0, 2 * h), code_h2(x0, 2 * h + 1), code_h2(x1, 2 * h),
                code_h2(x1, 2 * h + 1), bp[mt][0], bp[mt][1]);
        if (PV_LO)
          mma_f16(st.acc[mv], code_h2(x0, 2 * h), code_h2(x0, 2 * h + 1), code_h2(x1, 2 * h),
                  code_h2(x1, 2 * h + 1), bpl[PV_LO ? mt : 0][0], bpl[PV_LO ? mt : 0][1]);
      }
    }
  }
}

// Writes this warp's (m, l, y[c]) per head into shared memory.
// Quantized layout: channel 16g + 2mv + r with factor 2^24 4^-(2(mv&1)+r);
// residual layout: channel 16mv + g + 8r, no factor.
template <int NG, bool QUANT>
__device__ __forceinline__ void warp_store(WarpState<NG>& st, float* smrec, int lane) {
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int e = 0; e < NH; ++e) {
    float l = st.l[e], z = st.z[e];
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
      z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    st.l[e] = l;
    st.z[e] = z;
  }
#pragma unroll
  for (int e = 0; e < NH; ++e) {
    const int h = HILO ? t : 2 * t + e;
    if (h >= NG) continue;
    float* r = smrec + h * REC;
    if (g == 0) {
      r[0] = st.m[e];
      r[1] = st.l[e];
    }
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        float v = HILO ? st.acc[mv][2 * rr] + st.acc[mv][2 * rr + 1] : st.acc[mv][2 * rr + e];
        int ch;
        if (QUANT) {
          v = fmaf(v, code_unscale(2 * (mv & 1) + rr), st.z[e]);
          ch = 16 * g + 2 * mv + rr;
        } else {
          ch = 16 * mv + g + 8 * rr;
        }
        r[4 + ch] = v;
      }
    }
  }
}

// Merges the WARPS per-warp records in shared memory into one global record per head.
template <int NG>
__device__ __forceinline__ void cta_merge(const float* sm, float* out) {
  for (int i = threadIdx.x; i < NG * REC; i += THREADS) {
    const int h = i / REC, k = i % REC;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, sm[(w * NG + h) * REC]);
    float v;
    if (k == 0) {
      v = M;
    } else {
      v = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
          float mw = sm[(w * NG + h) * REC];
          if (mw != -INFINITY) v = fmaf(exp2f(mw - M), sm[(w * NG + h) * REC + k], v);
        }
      }
    }
    out[h * REC + k] = v;
  }
}

template <int NG, int EXTRA>
__device__ void run_quant(const DecArgs& a, int unit, int split, float* smrec) {
  const kvlc_cache& c = a.c;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr bool HILO = NG <= 4;
  // q fragments (fp16) for B column n = g
  uint32_t qh[8][2];
  {
    const int head = HILO ? (g >> 1) : g;
    const bool valid = head < NG;
    const uint16_t* qp = a.q + ((size_t)b * c.Hq + (size_t)kvh * NG + (valid ? head : 0)) * D + 4 * t;
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      uint2 raw = valid ? ldg2(qp + 16 * kt) : make_uint2(0u, 0u);
      float f0 = __uint_as_float(raw.x << 16), f1 = __uint_as_float(raw.x & 0xffff0000u);
      float f2 = __uint_as_float(raw.y << 16), f3 = __uint_as_float(raw.y & 0xffff0000u);
      qh[kt][0] = h2u(__floats2half2_rn(f0, f1));
      qh[kt][1] = h2u(__floats2half2_rn(f2, f3));
    }
  }
  WarpState<NG> st;
  st.init();
  const int n_ch = min(c.n_chunks[b], a.chunk_hi);
  const int lo = a.chunk_lo + split * a.cpw * WARPS;
  const int hi = min(n_ch, lo + a.cpw * WARPS);
  for (int ci = lo + warp; ci < hi; ci += WARPS)
    quant_chunk<NG, EXTRA>(c, (size_t)unit * c.max_chunks + ci, qh, st, lane);
  warp_store<NG, true>(st, smrec + warp * NG * REC, lane);
  __syncthreads();
  cta_merge<NG>(smrec, a.rec + ((size_t)unit * a.nrec + split) * NG * REC);
}

// Residual window half hf: ring slots [128 hf, 128 hf + 128), 32 per warp.
__device__ __forceinline__ int res_sigma(int r) {  // QK row -> slot offset within a 16-slot tile
  return r < 8 ? 2 * r - (r & 1) : 2 * (r - 8) - ((r - 8) & 1) + 2;
}

template <int NG>
__device__ void run_resid(const DecArgs& a, int unit, int hf, float* smrec) {
  const kvlc_cache& c = a.c;
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int start = c.res_start[b], len = c.res_len[b];
  const int base = 128 * hf + 32 * warp;
  WarpState<NG> st;
  st.init();
  auto live = [&](int slot) { return ((slot - start) & (SLOTS - 1)) < len; };
  bool any = false;
  for (int s = 0; s < 32; ++s) any |= live(base + s);
  if (any) {
    const uint16_t* kr = c.kres + (size_t)unit * SLOTS * D;
    const uint16_t* vr = c.vres + (size_t)unit * D * SLOTS;
    // q (bf16) B fragments: column n = g; channels 32kp + 8t + 4e + {0,1 | 2,3}
    uint32_t qb[4][4];
    {
      const int head = HILO ? (g >> 1) : g;
      const bool valid = HILO ? ((g & 1) == 0 && head < NG) : head < NG;
      const uint16_t* qp = a.q + ((size_t)b * c.Hq + (size_t)kvh * NG + (head < NG ? head : 0)) * D + 8 * t;
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {
        uint4 v = valid ? ldg4(qp + 32 * kp) : make_uint4(0u, 0u, 0u, 0u);
        qb[kp][0] = v.x;
        qb[kp][1] = v.y;
        qb[kp][2] = v.z;
        qb[kp][3] = v.w;
      }
    }
    float cr[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int j = 0; j < 4; ++j) cr[mt][j] = 0.f;
      const int sa = base + 16 * mt + res_sigma(g), sb = sa + 2;
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {
        uint4 ka = ldg4(kr + (size_t)sa * D + 32 * kp + 8 * t);
        uint4 kb = ldg4(kr + (size_t)sb * D + 32 * kp + 8 * t);
        mma_bf16(cr[mt], ka.x, kb.x, ka.y, kb.y, qb[kp][0], qb[kp][1]);
        mma_bf16(cr[mt], ka.z, kb.z, ka.w, kb.w, qb[kp][2], qb[kp][3]);
      }
    }
    // logits (log2 units), masking, softmax over the warp's 32 slots
    float cmax[NH];
#pragma unroll
    for (int e = 0; e < NH; ++e) cmax[e] = -INFINITY;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const bool lv = live(base + 16 * mt + res_sigma(g) + 2 * r);
#pragma unroll
        for (int e = 0; e < NH; ++e) {
          float v = HILO ? (cr[mt][2 * r] + cr[mt][2 * r + 1]) * C0 : cr[mt][2 * r + e] * C0;
          v = lv ? v : -INFINITY;
          cr[mt][2 * r + e] = v;
          cmax[e] = fmaxf(cmax[e], v);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < NH; ++e) {
      float m = cmax[e];
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
      st.m[e] = m;  // finite: at least one live slot in the warp
    }
    uint32_t bhi[2][2], blo[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (HILO) {
          float p = exp2f(cr[mt][2 * r] - st.m[0]);
          st.l[0] += p;
          __nv_bfloat16 hi = __float2bfloat16_rn(p);
          __nv_bfloat16 lo = __float2bfloat16_rn(p - __bfloat162float(hi));
          __nv_bfloat162 pk = __halves2bfloat162(hi, lo);
          bhi[mt][r] = movm_t(*reinterpret_cast<uint32_t*>(&pk));
        } else {
          float p0 = exp2f(cr[mt][2 * r] - st.m[0]);
          float p1 = exp2f(cr[mt][2 * r + 1] - st.m[1]);
          st.l[0] += p0;
          st.l[1] += p1;
          __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
          float2 hf2 = __bfloat1622float2(h);
          __nv_bfloat162 l2 = __floats2bfloat162_rn(p0 - hf2.x, p1 - hf2.y);
          bhi[mt][r] = movm_t(*reinterpret_cast<uint32_t*>(&h));
          blo[mt][r] = movm_t(*reinterpret_cast<uint32_t*>(&l2));
        }
      }
    }
    // PV: A = V^T rows (channels 16mv + g, +8), k = slots 16mt + 4t + {0,1 | 2,3}
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        uint2 va = ldg2(vr + (size_t)(16 * mv + g) * SLOTS + base + 16 * mt + 4 * t);
        uint2 vb = ldg2(vr + (size_t)(16 * mv + g + 8) * SLOTS + base + 16 * mt + 4 * t);
        mma_bf16(st.acc[mv], va.x, vb.x, va.y, vb.y, bhi[mt][0], bhi[mt][1]);
        if (!HILO) mma_bf16(st.acc[mv], va.x, vb.x, va.y, vb.y, blo[mt][0], blo[mt][1]);
      }
    }
  }
  warp_store<NG, false>(st, smrec + warp * NG * REC, lane);
  __syncthreads();
  cta_merge<NG>(smrec, a.rec + ((size_t)unit * a.nrec + a.nsq + hf) * NG * REC);
}

// C_n = S phi for CORR_ROWS rows of S (8 per warp).  Waits for phi_kernel.
template <int NG>
__device__ void run_corr(const DecArgs& a, int unit, int rb) {
  griddep_wait();
  const kvlc_cache& c = a.c;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t qh0 = (size_t)b * c.Hq + (size_t)kvh * NG;
  float ph[NG][8];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const float4* p = reinterpret_cast<const float4*>(a.phi + (qh0 + i) * RANK + lane * 8);
    float4 x = p[0], y = p[1];
    ph[i][0] = x.x; ph[i][1] = x.y; ph[i][2] = x.z; ph[i][3] = x.w;
    ph[i][4] = y.x; ph[i][5] = y.y; ph[i][6] = y.z; ph[i][7] = y.w;
  }
  const int row0 = rb * CORR_ROWS + warp * (CORR_ROWS / WARPS);
  float4 sr[CORR_ROWS / WARPS][2];
#pragma unroll
  for (int r = 0; r < CORR_ROWS / WARPS; ++r) {
    const float4* sp = reinterpret_cast<const float4*>(c.S + ((size_t)unit * D + row0 + r) * RANK + lane * 8);
    sr[r][0] = __ldg(sp);
    sr[r][1] = __ldg(sp + 1);
  }
#pragma unroll
  for (int r = 0; r < CORR_ROWS / WARPS; ++r) {
    const float s8[8] = {sr[r][0].x, sr[r][0].y, sr[r][0].z, sr[r][0].w,
                         sr[r][1].x, sr[r][1].y, sr[r][1].z, sr[r][1].w};
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      float v = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) v = fmaf(s8[k], ph[i][k], v);
      v = warp_sum(v);
      if (lane == i) a.corr[(qh0 + i) * (1 + D) + 1 + row0 + r] = v;
    }
  }
}

template <int NG, int EXTRA>
__global__ void __launch_bounds__(THREADS, 2) split_kernel(const DecArgs a) {
  __shared__ __align__(16) float smrec[WARPS * NG * REC];
  const int U = a.c.B * a.c.Hkv;
  int x = blockIdx.x;
  if (x < U * a.nsq) {
    run_quant<NG, EXTRA>(a, x / a.nsq, x % a.nsq, smrec);
    return;
  }
  x -= U * a.nsq;
  if (a.tail) {
    if (x < 2 * U) {
      run_resid<NG>(a, x / 2, x % 2, smrec);
      return;
    }
    x -= 2 * U;
    if (a.corr_on && x < U * CORR_CTAS) run_corr<NG>(a, x / CORR_CTAS, x % CORR_CTAS);
  }
}

// ------------------------------------------------------------ combine ----
// FWHT of 128 values, 4 per lane (channels 4 lane + e), unnormalised.
__device__ __forceinline__ void warp_fwht128(float (&x)[4], int lane) {
  float u0 = x[0] + x[1], u1 = x[0] - x[1], u2 = x[2] + x[3], u3 = x[2] - x[3];
  x[0] = u0 + u2;
  x[2] = u0 - u2;
  x[1] = u1 + u3;
  x[3] = u1 - u3;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float o = __shfl_xor_sync(0xffffffffu, x[e], k);
      x[e] = (lane & k) ? (o - x[e]) : (x[e] + o);
    }
  }
}

struct CombArgs {
  int B, Hq, NG, Hkv;
  const float* rec;  // decode: [U][nrec][NG][REC];  merge: [n][B][Hq][2+2D] with stride
  int nrec, nsq;     // decode mode
  int64_t rec_stride;
  const float* corr;  // [B][Hq][1+D] or null
  int literal;
  int out_fp32;
  void* out;          // [B][Hq][D] bf16 or f32 (final)
  float* rec_out;     // partial mode: [B][Hq][2+2D]
};

// Shared tail: apply the correction rule and produce out = (H num_rot + num_raw)/den.
__device__ __forceinline__ void finish(float M, float den, float (&nr)[4], float (&nw)[4],
                                       const float* corr, int literal, int lane, void* out,
                                       int out_fp32) {
  if (corr) {
    const float cd = corr[0];
    float cn[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) cn[e] = corr[1 + 4 * lane + e];
    bool any = cd != 0.f || cn[0] != 0.f || cn[1] != 0.f || cn[2] != 0.f || cn[3] != 0.f;
    any = __any_sync(0xffffffffu, any);
    if (any) {
      if (literal) {
#pragma unroll
        for (int e = 0; e < 4; ++e) nr[e] += cn[e];
        den += cd;
      } else if (M >= 0.f) {
        const float s = exp2f(-M);
#pragma unroll
        for (int e = 0; e < 4; ++e) nr[e] = fmaf(s, cn[e], nr[e]);
        den = fmaf(s, cd, den);
      } else {
        const float s = exp2f(M);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          nr[e] = fmaf(s, nr[e], cn[e]);
          nw[e] *= s;
        }
        den = fmaf(s, den, cd);
      }
    }
  }
  warp_fwht128(nr, lane);
  const float h = 0.08838834764831845f;  // fp32(1/sqrt(128))
  float r[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) r[e] = fmaf(nr[e], h, nw[e]) / den;
  if (out_fp32) {
    *reinterpret_cast<float4*>(static_cast<float*>(out) + 4 * lane) = make_float4(r[0], r[1], r[2], r[3]);
  } else {
    __nv_bfloat162 p0 = __floats2bfloat162_rn(r[0], r[1]), p1 = __floats2bfloat162_rn(r[2], r[3]);
    *reinterpret_cast<uint2*>(static_cast<uint16_t*>(out) + 4 * lane) =
        make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
  }
}

__global__ void __launch_bounds__(128) combine_kernel(const CombArgs a) {
  griddep_wait();
  const int gw = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gw >= a.B * a.Hq) return;
  const int b = gw / a.Hq, qh = gw % a.Hq, kvh = qh / a.NG, h = qh % a.NG;
  const int unit = b * a.Hkv + kvh;
  const float* base = a.rec + (size_t)unit * a.nrec * a.NG * REC + (size_t)h * REC;
  float M = -INFINITY;
  for (int r = 0; r < a.nrec; ++r) M = fmaxf(M, base[(size_t)r * a.NG * REC]);
  float nr[4] = {0.f, 0.f, 0.f, 0.f}, nw[4] = {0.f, 0.f, 0.f, 0.f}, den = 0.f;
  if (M != -INFINITY) {
    for (int r = 0; r < a.nrec; ++r) {
      const float* rr = base + (size_t)r * a.NG * REC;
      const float m = rr[0];
      if (m == -INFINITY) continue;
      const float w = exp2f(m - M);
      den = fmaf(w, rr[1], den);
      const float4 y = *reinterpret_cast<const float4*>(rr + 4 + 4 * lane);
      float* dst = r < a.nsq ? nr : nw;
      dst[0] = fmaf(w, y.x, dst[0]);
      dst[1] = fmaf(w, y.y, dst[1]);
      dst[2] = fmaf(w, y.z, dst[2]);
      dst[3] = fmaf(w, y.w, dst[3]);
    }
  }
  if (a.rec_out) {  // partial mode: (M, den, num_rot, num_raw), no correction
    float* o = a.rec_out + (size_t)gw * PREC;
    if (lane == 0) *reinterpret_cast<float4*>(o) = make_float4(M, den, 0.f, 0.f);
    *reinterpret_cast<float4*>(o + 4 + 4 * lane) = make_float4(nr[0], nr[1], nr[2], nr[3]);
    *reinterpret_cast<float4*>(o + 4 + D + 4 * lane) = make_float4(nw[0], nw[1], nw[2], nw[3]);
    return;
  }
  void* o = a.out_fp32 ? (void*)(static_cast<float*>(a.out) + (size_t)gw * D)
                       : (void*)(static_cast<uint16_t*>(a.out) + (size_t)gw * D);
  finish(M, den, nr, nw, a.corr ? a.corr + (size_t)gw * (1 + D) : nullptr, a.literal, lane, o, a.out_fp32);
}

// LSE merge of n device records (m, l, y_rot, y_raw) + correction -> out.
__global__ void __launch_bounds__(128) merge_records_kernel(const float* __restrict__ recs, int n,
                                                            int64_t stride, const float* __restrict__ corr,
                                                            int BH, int literal, int out_fp32,
                                                            void* __restrict__ out) {
  const int gw = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gw >= BH) return;
  float M = -INFINITY;
  for (int r = 0; r < n; ++r) M = fmaxf(M, recs[r * stride + (size_t)gw * PREC]);
  float nr[4] = {0.f, 0.f, 0.f, 0.f}, nw[4] = {0.f, 0.f, 0.f, 0.f}, den = 0.f;
  if (M != -INFINITY) {
    for (int r = 0; r < n; ++r) {
      const float* rr = recs + r * stride + (size_t)gw * PREC;
      if (rr[0] == -INFINITY) continue;
      const float w = exp2f(rr[0] - M);
      den = fmaf(w, rr[1], den);
      const float4 y = *reinterpret_cast<const float4*>(rr + 4 + 4 * lane);
      const float4 z = *reinterpret_cast<const float4*>(rr + 4 + D + 4 * lane);
      nr[0] = fmaf(w, y.x, nr[0]); nr[1] = fmaf(w, y.y, nr[1]);
      nr[2] = fmaf(w, y.z, nr[2]); nr[3] = fmaf(w, y.w, nr[3]);
      nw[0] = fmaf(w, z.x, nw[0]); nw[1] = fmaf(w, z.y, nw[1]);
      nw[2] = fmaf(w, z.z, nw[2]); nw[3] = fmaf(w, z.w, nw[3]);
    }
  }
  void* o = out_fp32 ? (void*)(static_cast<float*>(out) + (size_t)gw * D)
                     : (void*)(static_cast<uint16_t*>(out) + (size_t)gw * D);
  finish(M, den, nr, nw, corr ? corr + (size_t)gw * (1 + D) : nullptr, literal, lane, o, out_fp32);
}

// ------------------------------------------------------------- host ----
struct Plan {
  int NG, U, nsq, cpw, nrec, corr_on;
  size_t phi_off, corr_off, rec_off, total;
};

int plan_for(const kvlc_cache* c, const kvlc_decode_opts* o, int chunk_lo, int chunk_hi, int tail,
             bool corr_on, Plan& p) {
  KVLC_REQUIRE(c && c->B >= 1 && c->Hkv >= 1 && c->Hq % c->Hkv == 0 && c->Hq / c->Hkv <= 8,
               "bad cache dims");
  p.NG = c->Hq / c->Hkv;
  p.U = c->B * c->Hkv;
  int maxc = o && o->max_chunks_hint > 0 ? o->max_chunks_hint : c->max_chunks;
  int span = std::max(0, std::min(maxc, chunk_hi) - chunk_lo);
  int cpw = o && o->chunks_per_split > 0 ? o->chunks_per_split : 0;
  if (cpw == 0) {
    // aim for ~16 warps of work per SM across the grid
    long long warps_wanted = 148LL * 16;
    long long chunks = (long long)p.U * std::max(span, 1);
    cpw = (int)std::max(1LL, std::min(16LL, chunks / warps_wanted));
  }
  p.cpw = cpw;
  p.nsq = std::max(1, (span + cpw * WARPS - 1) / (cpw * WARPS));
  p.corr_on = corr_on && tail ? 1 : 0;
  p.nrec = p.nsq + (tail ? 2 : 0);
  size_t BH = (size_t)c->B * c->Hq;
  p.phi_off = 0;
  p.corr_off = align_up(BH * RANK * sizeof(float));
  p.rec_off = p.corr_off + align_up(BH * (1 + D) * sizeof(float));
  p.total = p.rec_off + align_up((size_t)p.U * p.nrec * p.NG * REC * sizeof(float));
  return KVLC_OK;
}

template <int NG>
int launch_ng(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q, const Plan& p,
              char* ws, int chunk_lo, int chunk_hi, int tail, float* corr_ext, int literal,
              int out_fp32, void* out, float* rec_out, cudaStream_t s) {
  float* phi = reinterpret_cast<float*>(ws + p.phi_off);
  float* corr = corr_ext ? corr_ext : reinterpret_cast<float*>(ws + p.corr_off);
  float* rec = reinterpret_cast<float*>(ws + p.rec_off);
  if (p.corr_on) {
    phi_kernel<NG><<<p.U, 256, 0, s>>>(*c, ad->w1q, ad->w2q, q, phi, corr);
    int rc = check_launch("phi");
    if (rc) return rc;
  }
  DecArgs a{};
  a.c = *c;
  a.q = q;
  a.phi = phi;
  a.corr = corr;
  a.rec = rec;
  a.nsq = p.nsq;
  a.cpw = p.cpw;
  a.chunk_lo = chunk_lo;
  a.chunk_hi = chunk_hi;
  a.tail = tail;
  a.corr_on = p.corr_on;
  a.nrec = p.nrec;
  int grid = p.U * p.nsq + (tail ? 2 * p.U + (p.corr_on ? p.U * CORR_CTAS : 0) : 0);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = p.corr_on ? 1 : 0;
  if (NG <= 4) {
    KVLC_CUDA(cudaLaunchKernelEx(&cfg, split_kernel<NG, 0>, a));
  } else {
    // precision passes for > 4 heads per group (see quant_chunk); KVLC_EXTRA overrides (tuning)
    static const int extra = [] {
      const char* e = getenv("KVLC_EXTRA");
      return e ? atoi(e) & 3 : 3;
    }();
    switch (extra) {
      case 0: KVLC_CUDA(cudaLaunchKernelEx(&cfg, split_kernel<NG, 0>, a)); break;
      case 1: KVLC_CUDA(cudaLaunchKernelEx(&cfg, split_kernel<NG, 1>, a)); break;
      case 2: KVLC_CUDA(cudaLaunchKernelEx(&cfg, split_kernel<NG, 2>, a)); break;
      default: KVLC_CUDA(cudaLaunchKernelEx(&cfg, split_kernel<NG, 3>, a)); break;
    }
  }
  CombArgs ca{};
  ca.B = c->B;
  ca.Hq = c->Hq;
  ca.NG = NG;
  ca.Hkv = c->Hkv;
  ca.rec = rec;
  ca.nrec = p.nrec;
  ca.nsq = p.nsq;
  ca.corr = p.corr_on ? corr : nullptr;
  ca.literal = literal;
  ca.out_fp32 = out_fp32;
  ca.out = out;
  ca.rec_out = rec_out;
  cudaLaunchConfig_t cfg2{};
  cfg2.gridDim = dim3((c->B * c->Hq + 3) / 4);
  cfg2.blockDim = dim3(128);
  cfg2.stream = s;
  cfg2.attrs = attr;
  cfg2.numAttrs = 1;
  KVLC_CUDA(cudaLaunchKernelEx(&cfg2, combine_kernel, ca));
  return check_launch("decode");
}

int launch(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q, const Plan& p, char* ws,
           int chunk_lo, int chunk_hi, int tail, float* corr_ext, int literal, int out_fp32, void* out,
           float* rec_out, cudaStream_t s) {
  switch (p.NG) {
#define KVLC_NG_CASE(n) \
  case n:               \
    return launch_ng<n>(c, ad, q, p, ws, chunk_lo, chunk_hi, tail, corr_ext, literal, out_fp32, out, rec_out, s);
    KVLC_NG_CASE(1)
    KVLC_NG_CASE(2)
    KVLC_NG_CASE(3)
    KVLC_NG_CASE(4)
    KVLC_NG_CASE(5)
    KVLC_NG_CASE(6)
    KVLC_NG_CASE(7)
    KVLC_NG_CASE(8)
#undef KVLC_NG_CASE
    default:
      return fail(KVLC_EINVAL, "GQA group %d not supported (1..8)", p.NG);
  }
}

bool adapter_active(const kvlc_adapter* ad) {
  return ad != nullptr && ad->enabled && ad->w1q && ad->w2q;
}

}  // namespace
}  // namespace kvlc

using namespace kvlc;

extern "C" {

size_t kvlc_decode_workspace(const kvlc_cache* c, const kvlc_decode_opts* o) {
  Plan p;
  if (!c || plan_for(c, o, 0, 1 << 30, 1, true, p)) return 0;
  return p.total;
}

int kvlc_decode(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q, void* out,
                const kvlc_decode_opts* o, void* ws, size_t ws_bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(q && out, "null query / output");
  Plan p;
  int rc = plan_for(c, o, 0, 1 << 30, 1, adapter_active(ad), p);
  if (rc) return rc;
  KVLC_REQUIRE(ws && ws_bytes >= p.total, "decode workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
  return launch(c, ad, q, p, static_cast<char*>(ws), 0, 1 << 30, 1, nullptr, o ? o->literal : 0,
                o ? o->out_fp32 : 0, out, nullptr, as_stream(stream));
}

int kvlc_decode_partial(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q,
                        int32_t chunk_lo, int32_t chunk_hi, int32_t include_tail, float* rec,
                        float* corr, const kvlc_decode_opts* o, void* ws, size_t ws_bytes,
                        void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(q && rec, "null query / record buffer");
  KVLC_REQUIRE(chunk_lo >= 0 && chunk_hi >= chunk_lo, "bad chunk window [%d, %d)", chunk_lo, chunk_hi);
  KVLC_REQUIRE(!include_tail || !adapter_active(ad) || corr, "tail owner needs a correction buffer");
  Plan p;
  int rc = plan_for(c, o, chunk_lo, chunk_hi, include_tail ? 1 : 0, adapter_active(ad), p);
  if (rc) return rc;
  KVLC_REQUIRE(ws && ws_bytes >= p.total, "decode workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
  if (include_tail && corr && !p.corr_on)
    KVLC_CUDA(cudaMemsetAsync(corr, 0, (size_t)c->B * c->Hq * (1 + D) * sizeof(float), as_stream(stream)));
  return launch(c, ad, q, p, static_cast<char*>(ws), chunk_lo, chunk_hi, include_tail ? 1 : 0, corr,
                0, 0, nullptr, rec, as_stream(stream));
}

int kvlc_merge_records(const float* recs, int32_t n_rec, int64_t rec_stride, const float* corr,
                       int32_t B, int32_t Hq, int32_t literal, int32_t out_fp32, void* out,
                       void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(recs && out && n_rec >= 1 && B >= 1 && Hq >= 1, "bad merge arguments");
  const int BH = B * Hq;
  merge_records_kernel<<<(BH + 3) / 4, 128, 0, as_stream(stream)>>>(recs, n_rec, rec_stride, corr, BH,
                                                                     literal, out_fp32, out);
  return check_launch("merge_records");
}

}  // extern "C"
