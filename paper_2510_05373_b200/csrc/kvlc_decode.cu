// Fused KVLinC decode for the batched serving cache (d = G = 128, 2-bit).
//
// Reference: decode_step_blocked (attention.py:197-276) = Algorithm 1
// (PAPER.md:172-199): per-block fp32 scores / max / exp / partial numerators
// over the quantized history, one extra full-precision block for the
// residual window, the phi_q(q)·S / phi_q(q)·P correction folded with the
// e^{-M}-consistent rule (_reduce_blocks, attention.py:158-194), the inverse
// Hadamard rotation of the quantized numerator and the final divide.
//
// Kernels (one decode step = 2 launches, PDL-chained):
//   split_kernel    per CTA task, selected by blockIdx:
//                   * correction (first, one per unit): phi_q of the unit's
//                     query heads, C_d = P phi, C_n = S phi (attention.py:224-231)
//                   * quantized split: chunks of one (b, kv-head) unit, GQA
//                     heads batched on the MMA N dimension, 2-bit codes turned
//                     into fp16 MMA operands by one LOP3 each (exact subnormal
//                     values c * 4^j * 2^-24), scales folded into q / p
//                     (hi+lo fp16 split when the group has <= 4 heads)
//                     (kvlc_quant.cuh)
//                   * residual half: bf16 ring window, masked
//   combine_kernel  per (b, q-head): the LSE merge of the unit's records +
//                   correction, the warp FWHT (H^T = H) and the divide.  Plans
//                   with more than CMB_MAXREC records per unit fuse it instead
//                   into the last arriving CTA of each unit (arrival counters).
//
// Online-softmax state is kept in log2 units (logit * log2 e); the sign of the
// global max, which selects the correction branch, is unit independent.
#include "kvlc_common.cuh"
#include "kvlc_tc.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace kvlc {
namespace {

constexpr int D = KVLC_D;
constexpr int SLOTS = KVLC_SLOTS;
constexpr int RANK = KVLC_RANK;
constexpr int HALF = RANK / 2;
constexpr int WARPS = 4;
constexpr int THREADS = WARPS * 32;
constexpr int REC = 4 + D;  // record: m (log2 units), l, pad, pad, y[D] (16-byte aligned y)
constexpr int PREC = 4 + 2 * D;  // device-partial record: m, l, pad, pad, y_rot[D], y_raw[D]
constexpr float C0 = 0.12751743074173226f;  // log2(e) / sqrt(128)

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
// half2 of fp16 subnormals (c_lo * 4^(j+1) * 2^-24, c_hi * 4^(j+1) * 2^-24) from a stored
// (rotated, frag_store) word: bytes 0 / 2 of the unrotated word; code_hi(x) brings bytes 1 / 3
__device__ __forceinline__ uint32_t code_h2(uint32_t x, int j) { return x & (0x000C000Cu << (2 * j)); }
__device__ __forceinline__ uint32_t code_hi(uint32_t x) { return __funnelshift_r(x, x, 8); }

// 2^24 * 4^-(j+1)
__device__ __forceinline__ constexpr float code_unscale(int j) {
  return j == 0 ? 4194304.f : (j == 1 ? 1048576.f : (j == 2 ? 262144.f : 65536.f));
}

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n"); }

struct DecArgs {
  kvlc_cache c;
  const uint16_t* q;      // [B][Hq][D] bf16
  const float* w1q;       // [Hkv][D][HALF] fp32 (phi_q weights, adapter.py:91-93)
  const float* w2q;
  float* corr;            // [2][B][Hq][1 + D]: (C_d, C_n) partials of the two feature halves
  size_t corr_half;       // B * Hq * (1 + D)
  float* corr_ext;        // partial mode: the caller's [B][Hq][1 + D] (the halves' sum)
  int corr_split;         // correction CTAs per unit: 1 (run_corr_unit) or 2 (run_corr halves)
  float* rec;             // [U][nrec][NG][REC]
  int nsq;                // quantized split CTAs per unit
  int cpc;                // chunks per quantized-split CTA
  int chunk_lo, chunk_hi; // global chunk window (split-KV across devices)
  int tail;               // include residual window + correction rows
  int corr_on;            // adapter active
  int nrec;               // records per unit = nsq + 2*tail
  // fused LSE combine: the last CTA of a unit merges its records
  uint32_t* done;         // [U] arrival counters (zeroed before the launch, self-cleaning)
  int literal;
  int out_fp32;
  void* out;              // [B][Hq][D] bf16 / f32 (final output)
  float* rec_out;         // partial mode: [B][Hq][PREC] (split-KV across devices)
  int sep_combine;        // 1: the combine is combine_kernel, PDL-chained (no arrival counters)
  int tail_fused;         // correction half h and residual half h of a unit in one task
  int rps;                // records per quantized split: 1 (CTA-merged) or 4 (one per warp)
  int qrec;               // quantized records per unit (nsq * rps); residual records follow
  uint32_t* queue;        // persistent split grid: task counter (zero between launches), or null
  int ntask;              // tasks of the split grid
};

#ifdef KVLC_TRACE
// per-CTA timeline (tools/trace_decode.py): globaltimer at entry, before the arrival
// atomic and at exit, task kind (0 correction, 1 split, 2 residual), SM id
constexpr int DT_MAX = 8192;
__device__ unsigned long long g_dtrace[DT_MAX][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}
#define DT_STAMP(i, v) \
  do { if (threadIdx.x == 0 && blockIdx.x < DT_MAX) g_dtrace[blockIdx.x][i] = (v); } while (0)
// phase stamps inside a task (tools/trace_decode.py prints them per task kind)
__device__ unsigned long long g_dphase[DT_MAX][4];
#define PH_STAMP(i) \
  do { if (threadIdx.x == 0 && blockIdx.x < DT_MAX) g_dphase[blockIdx.x][i] = gtimer(); } while (0)
#else
#define PH_STAMP(i) do { } while (0)
#define DT_STAMP(i, v) do { } while (0)
#endif

#include "kvlc_quant.cuh"
#include "kvlc_quant_wpc.cuh"

// Residual window half hf: ring slots [128 hf, 128 hf + 128), 32 per warp.
__device__ __forceinline__ int res_sigma(int r) {  // QK row -> slot offset within a 16-slot tile
  return r < 8 ? 2 * r - (r & 1) : 2 * (r - 8) - ((r - 8) & 1) + 2;
}

template <int NG>
__device__ __forceinline__ void run_resid(const DecArgs& a, int unit, int hf, float* smrec) {
  const kvlc_cache& c = a.c;
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  griddep_wait();  // the ring and its window may come from a programmatic-launch predecessor (append)
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
      st.mt[e] = m;
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
  cta_merge<NG>(smrec, a.rec + ((size_t)unit * a.nrec + a.qrec + hf) * NG * REC);
}

// Correction of one unit by one CTA (both feature halves; used when the splits and these
// CTAs fit one wave, see corr_split): phi_q of the unit's NG query heads
// (feature_map, adapter.py:80-88: thread t owns feature t of each half, W columns
// read from L2 8 channels per round trip), then C_d = P . phi and C_n = S phi for all
// 128 rows of S (8 / 4 rows per warp per pass, lanes across the 256 features).  These
// CTAs come first in the grid, so their S stream overlaps the code stream.
template <int NG>
__device__ __forceinline__ void run_corr_unit(const DecArgs& a, int unit, float* smf) {
  static_assert(HALF == THREADS, "one feature of each half per thread");
  const kvlc_cache& c = a.c;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const size_t qh0 = (size_t)b * c.Hq + (size_t)kvh * NG;
  constexpr int PART = WARPS * 2 * NG * HALF;          // per-warp partial z of both halves
  constexpr int REG = PART > NG * RANK ? PART : NG * RANK;
  float* qs = smf;                    // [NG][D]
  float* part = qs + NG * D;          // [WARPS][2][NG][HALF], then phs [NG][RANK] (aliased)
  float* phs = part;
  float* red = part + REG;            // [WARPS][2 NG]
  float* stat = red + WARPS * 2 * NG; // [2 NG]
  // the unit's S rows into L2 (row t, 1 KB) while phi_q is computed (r02, as run_corr)
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], 1024;\n" ::"l"(c.S + ((size_t)unit * D + t) * RANK)
               : "memory");
  // z = q W_h for both halves: warp w takes channels 32w..32w+31, lane l features 4l..4l+3
  // (16-B loads of W rows, 16 in flight), the warps' partial sums meet in shared memory
  constexpr int PB = 16;
  float4 w[PB];
  const float4* const W1 = reinterpret_cast<const float4*>(a.w1q + ((size_t)kvh * D + 32 * warp) * HALF) + lane;
  const float4* const W2 = reinterpret_cast<const float4*>(a.w2q + ((size_t)kvh * D + 32 * warp) * HALF) + lane;
#pragma unroll
  for (int k = 0; k < PB; ++k) w[k] = __ldg(W1 + k * (HALF / 4));   // L2-resident: before the wait
  griddep_wait();  // q may come from a programmatic-launch predecessor (kvlc_stage_input)
  {  // all NG loads in flight before the shared-memory stores
    uint16_t qv[NG];
#pragma unroll
    for (int i = 0; i < NG; ++i) qv[i] = __ldg(a.q + (qh0 + i) * D + t);
#pragma unroll
    for (int i = 0; i < NG; ++i) qs[i * D + t] = bf2f(qv[i]);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {  // (half, channel slice) rounds of PB rows
    const int hh = r >> 1, c0 = 32 * warp + PB * (r & 1);
    float zz[NG][4];
#pragma unroll
    for (int i = 0; i < NG; ++i) zz[i][0] = zz[i][1] = zz[i][2] = zz[i][3] = 0.f;
#pragma unroll
    for (int k = 0; k < PB; ++k) {
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        const float x = qs[i * D + c0 + k];
        zz[i][0] = fmaf(x, w[k].x, zz[i][0]);
        zz[i][1] = fmaf(x, w[k].y, zz[i][1]);
        zz[i][2] = fmaf(x, w[k].z, zz[i][2]);
        zz[i][3] = fmaf(x, w[k].w, zz[i][3]);
      }
    }
    if (r + 1 < 4) {
      const int h2 = (r + 1) >> 1, o2 = PB * ((r + 1) & 1);
#pragma unroll
      for (int k = 0; k < PB; ++k) w[k] = __ldg((h2 ? W2 : W1) + (o2 + k) * (HALF / 4));
    }
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      float4* dst = reinterpret_cast<float4*>(part + ((warp * 2 + hh) * NG + i) * HALF + 4 * lane);
      if (r & 1) {
        float4 o = *dst;
        o.x += zz[i][0]; o.y += zz[i][1]; o.z += zz[i][2]; o.w += zz[i][3];
        *dst = o;
      } else {
        *dst = make_float4(zz[i][0], zz[i][1], zz[i][2], zz[i][3]);
      }
    }
  }
  __syncthreads();
  float z[2][NG];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      float v = part[(h * NG + i) * HALF + t];
#pragma unroll
      for (int w2 = 1; w2 < WARPS; ++w2) v += part[((w2 * 2 + h) * NG + i) * HALF + t];
      z[h][i] = v;
    }
  // max-shifted softmax of each half (linalg.py:38-47)
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const float m = warp_max(z[h][i]);
      if (lane == 0) red[warp * 2 * NG + h * NG + i] = m;
    }
  __syncthreads();
  if (t < 2 * NG) {
    float m = red[t];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) m = fmaxf(m, red[w * 2 * NG + t]);
    stat[t] = m;
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < NG; ++i) z[h][i] = expf(z[h][i] - stat[h * NG + i]);
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      const float sm_ = warp_sum(z[h][i]);
      if (lane == 0) red[warp * 2 * NG + h * NG + i] = sm_;
    }
  __syncthreads();
  if (t < 2 * NG) {
    float sm_ = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) sm_ += red[w * 2 * NG + t];
    stat[t] = sm_;
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < NG; ++i) phs[i * RANK + h * HALF + t] = z[h][i] / stat[h * NG + i];
  __syncthreads();

  float ph[NG][8];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const float4 x = *reinterpret_cast<const float4*>(phs + i * RANK + lane * 8);
    const float4 y = *reinterpret_cast<const float4*>(phs + i * RANK + lane * 8 + 4);
    ph[i][0] = x.x; ph[i][1] = x.y; ph[i][2] = x.z; ph[i][3] = x.w;
    ph[i][4] = y.x; ph[i][5] = y.y; ph[i][6] = y.z; ph[i][7] = y.w;
  }
  if (warp == 0) {  // C_d = P . phi_q (attention.py:228)
    const float4* pp = reinterpret_cast<const float4*>(c.P + (size_t)unit * RANK + lane * 8);
    const float4 x = __ldg(pp), y = __ldg(pp + 1);
    const float p8[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      float v = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) v = fmaf(p8[k], ph[i][k], v);
      v = warp_sum(v);
      if (lane == 0) a.corr[(qh0 + i) * (1 + D)] = v;
    }
  }
  // C_n = S phi (attention.py:227): per pass a warp takes RPW rows; per-lane partial
  // dots, then one reduce-scatter per 32 values (lane L ends with value L's total)
  constexpr int RPW = NG > 4 ? 4 : 8;  // rows per warp per pass (register budget at 8 heads)
  constexpr int NV = RPW * NG;
  constexpr int NB = (NV + 31) / 32;
#pragma unroll 1
  for (int row0 = warp * RPW; row0 < D; row0 += WARPS * RPW) {
    float4 sr[RPW][2];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const float4* sp = reinterpret_cast<const float4*>(c.S + ((size_t)unit * D + row0 + r) * RANK + lane * 8);
      sr[r][0] = __ldg(sp);
      sr[r][1] = __ldg(sp + 1);
    }
    float vals[NB * 32];
#pragma unroll
    for (int n = 0; n < NB * 32; ++n) vals[n] = 0.f;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const float s8[8] = {sr[r][0].x, sr[r][0].y, sr[r][0].z, sr[r][0].w,
                           sr[r][1].x, sr[r][1].y, sr[r][1].z, sr[r][1].w};
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        float v = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) v = fmaf(s8[k], ph[i][k], v);
        vals[r * NG + i] = v;
      }
    }
#pragma unroll
    for (int blk = 0; blk < NB; ++blk) {
      float* x = vals + 32 * blk;
#pragma unroll
      for (int sft = 16; sft >= 1; sft >>= 1) {
        const bool upper = lane & sft;
#pragma unroll
        for (int k = 0; k < sft; ++k) {
          const float send = upper ? x[k] : x[k + sft];
          const float keep = upper ? x[k + sft] : x[k];
          x[k] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
        }
      }
      const int n = 32 * blk + lane;
      if (n < NV) {
        const int r = n / NG, i = n % NG;
        a.corr[(qh0 + i) * (1 + D) + 1 + row0 + r] = x[0];
      }
    }
  }
}

// The half's C_d = P_h . phi_h and C_n = S[:, h] phi_h partials (attention.py:227-228) from
// phi_h in shared memory (phs [NG][HALF]).
template <int NG>
__device__ __forceinline__ void corr_half_dots(const DecArgs& a, int unit, int h, const float* phs, float* corr,
                                               size_t qh0, int warp, int lane) {
  const kvlc_cache& c = a.c;
  float ph[NG][4];  // features 4 lane .. 4 lane + 3 of the half
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const float4 x = *reinterpret_cast<const float4*>(phs + i * HALF + lane * 4);
    ph[i][0] = x.x; ph[i][1] = x.y; ph[i][2] = x.z; ph[i][3] = x.w;
  }
  if (warp == 0) {  // C_d partial = P_h . phi_h (attention.py:228)
    const float4 x = __ldg(reinterpret_cast<const float4*>(c.P + (size_t)unit * RANK + h * HALF + lane * 4));
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      float v = x.x * ph[i][0];
      v = fmaf(x.y, ph[i][1], v);
      v = fmaf(x.z, ph[i][2], v);
      v = fmaf(x.w, ph[i][3], v);
      v = warp_sum(v);
      if (lane == 0) corr[(qh0 + i) * (1 + D)] = v;
    }
  }
  // C_n partial = S[:, h] phi_h (attention.py:227): per pass a warp takes RPW rows; per-lane
  // partial dots, then one reduce-scatter per 32 values (lane L ends with value L's total)
  constexpr int RPW = NG > 4 ? 8 : 16;  // rows per warp per pass (register budget at 8 heads)
  constexpr int NV = RPW * NG;
  constexpr int NB = (NV + 31) / 32;
#pragma unroll 1
  for (int row0 = warp * RPW; row0 < D; row0 += WARPS * RPW) {
    float4 sr[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
      sr[r] = __ldg(reinterpret_cast<const float4*>(c.S + ((size_t)unit * D + row0 + r) * RANK + h * HALF + lane * 4));
    float vals[NB * 32];
#pragma unroll
    for (int n = 0; n < NB * 32; ++n) vals[n] = 0.f;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        float v = sr[r].x * ph[i][0];
        v = fmaf(sr[r].y, ph[i][1], v);
        v = fmaf(sr[r].z, ph[i][2], v);
        v = fmaf(sr[r].w, ph[i][3], v);
        vals[r * NG + i] = v;
      }
    }
#pragma unroll
    for (int blk = 0; blk < NB; ++blk) {
      float* x = vals + 32 * blk;
#pragma unroll
      for (int sft = 16; sft >= 1; sft >>= 1) {
        const bool upper = lane & sft;
#pragma unroll
        for (int k = 0; k < sft; ++k) {
          const float send = upper ? x[k] : x[k + sft];
          const float keep = upper ? x[k + sft] : x[k];
          x[k] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
        }
      }
      const int n = 32 * blk + lane;
      if (n < NV) {
        const int r = n / NG, i = n % NG;
        corr[(qh0 + i) * (1 + D) + 1 + row0 + r] = x[0];
      }
    }
  }
}

// Correction of one unit, feature half h (attention.py:224-231): phi_q of the unit's NG
// query heads over half h (feature_map, adapter.py:80-88: the softmax is per half, so the
// halves are independent), then the half's partial C_d = P_h . phi_h and C_n = S[:, h] phi_h.
// Latency, not work, sets these CTAs' time (r02 traces: ~10 us, S and W load rounds), so:
//   * the half's S columns are prefetched into L2 at CTA start (one 512-B bulk prefetch per
//     row), before the predecessor grid is waited for;
//   * z = q W_h splits the channels over the warps (warp w: channels 32w..32w+31, lane l:
//     features 4l..4l+3, 16-B loads of W rows, two rounds of 16 in flight instead of four
//     rounds of 32 scalar loads), the 4 warps' partial sums meet in shared memory;
//   * C_n takes two passes of 16 rows per warp (groups of <= 4 heads).
// Two CTAs per unit halve the longest task of the grid; the combine adds the halves.  These
// CTAs come first in the grid, so their S stream overlaps the codes.
template <int NG>
__device__ __forceinline__ void run_corr(const DecArgs& a, int unit, int h, float* smf) {
  static_assert(HALF == THREADS, "one feature of the half per thread");
  const kvlc_cache& c = a.c;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const size_t qh0 = (size_t)b * c.Hq + (size_t)kvh * NG;
  float* corr = a.corr + (size_t)h * a.corr_half;
  float* qs = smf;                      // [NG][D]
  float* part = qs + NG * D;            // [WARPS][NG][HALF] partial z, then phs [NG][HALF]
  float* red = part + WARPS * NG * HALF;  // [WARPS][NG]
  float* stat = red + WARPS * NG;       // [NG]
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;\n" ::"l"(c.S + ((size_t)unit * D + t) * RANK + h * HALF)
               : "memory");
  const float4* W = reinterpret_cast<const float4*>((h ? a.w2q : a.w1q) + ((size_t)kvh * D + 32 * warp) * HALF) + lane;
  constexpr int PB = 16;  // W rows (16-B loads) in flight per thread
  float4 w[PB];
#pragma unroll
  for (int k = 0; k < PB; ++k) w[k] = __ldg(W + k * (HALF / 4));  // L2-resident: before the wait
  griddep_wait();  // q may come from a programmatic-launch predecessor (kvlc_stage_input)
  PH_STAMP(0);
  {  // all NG loads in flight before the shared-memory stores
    uint16_t qv[NG];
#pragma unroll
    for (int i = 0; i < NG; ++i) qv[i] = __ldg(a.q + (qh0 + i) * D + t);
#pragma unroll
    for (int i = 0; i < NG; ++i) qs[i * D + t] = bf2f(qv[i]);
  }
  __syncthreads();
  PH_STAMP(1);
  float z[NG][4];
#pragma unroll
  for (int i = 0; i < NG; ++i) z[i][0] = z[i][1] = z[i][2] = z[i][3] = 0.f;
#pragma unroll
  for (int r = 0; r < 32 / PB; ++r) {
#pragma unroll
    for (int k = 0; k < PB; ++k) {
      const int ch = 32 * warp + PB * r + k;
#pragma unroll
      for (int i = 0; i < NG; ++i) {
        const float x = qs[i * D + ch];
        z[i][0] = fmaf(x, w[k].x, z[i][0]);
        z[i][1] = fmaf(x, w[k].y, z[i][1]);
        z[i][2] = fmaf(x, w[k].z, z[i][2]);
        z[i][3] = fmaf(x, w[k].w, z[i][3]);
      }
    }
    if (r + 1 < 32 / PB) {
#pragma unroll
      for (int k = 0; k < PB; ++k) w[k] = __ldg(W + (PB * (r + 1) + k) * (HALF / 4));
    }
  }
#pragma unroll
  for (int i = 0; i < NG; ++i)
    *reinterpret_cast<float4*>(part + (warp * NG + i) * HALF + 4 * lane) = make_float4(z[i][0], z[i][1], z[i][2], z[i][3]);
  __syncthreads();
  float zf[NG];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    zf[i] = part[i * HALF + t];
#pragma unroll
    for (int w2 = 1; w2 < WARPS; ++w2) zf[i] += part[(w2 * NG + i) * HALF + t];
  }
  // max-shifted softmax of the half (linalg.py:38-47)
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const float m = warp_max(zf[i]);
    if (lane == 0) red[warp * NG + i] = m;
  }
  __syncthreads();
  if (t < NG) {
    float m = red[t];
#pragma unroll
    for (int w2 = 1; w2 < WARPS; ++w2) m = fmaxf(m, red[w2 * NG + t]);
    stat[t] = m;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NG; ++i) zf[i] = expf(zf[i] - stat[i]);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    const float sm_ = warp_sum(zf[i]);
    if (lane == 0) red[warp * NG + i] = sm_;
  }
  __syncthreads();
  if (t < NG) {
    float sm_ = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < WARPS; ++w2) sm_ += red[w2 * NG + t];
    stat[t] = sm_;
  }
  __syncthreads();
  float* phs = part;  // every thread has read its partial sums (barriers above)
#pragma unroll
  for (int i = 0; i < NG; ++i) phs[i * HALF + t] = zf[i] / stat[i];
  __syncthreads();
  PH_STAMP(2);
  corr_half_dots<NG>(a, unit, h, phs, corr, qh0, warp, lane);
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
      x[e] = fmaf(x[e], (lane & k) ? -1.f : 1.f, o);  // o - x or x + o, one FFMA (exact)
    }
  }
}

// Shared tail: apply the correction rule and produce out = (H num_rot + num_raw)/den.
// num/den are expressed in the frame 2^-M (M = max of the records' reference
// points); Mt is the true global logit max (the reference's M, attention.py:172-175).
// Consistent correction: C enters as the m = 0 partial, i.e. scaled by 2^-M when
// M >= 0, else the blocks are scaled by 2^M (attention.py:190-194); both are the
// same value as the reference's e^-M_true form.  Literal mode adds C unscaled in
// the true-max frame (attention.py:188-189).
// corr: nullptr, or {C_d, C_n[4*lane .. 4*lane+3]} of this lane.
__device__ __forceinline__ void finish(float M, float Mt, float den, float (&nr)[4], float (&nw)[4],
                                       const float* corr, int literal, int lane, void* out,
                                       int out_fp32) {
  if (corr) {
    const float cd = corr[0];
    float cn[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) cn[e] = corr[1 + e];
    bool any = cd != 0.f || cn[0] != 0.f || cn[1] != 0.f || cn[2] != 0.f || cn[3] != 0.f;
    any = __any_sync(0xffffffffu, any);
    if (any) {
      if (literal) {
        const float s = M == -INFINITY ? 0.f : exp2f(M - Mt);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          nr[e] = fmaf(s, nr[e], cn[e]);
          nw[e] *= s;
        }
        den = fmaf(s, den, cd);
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

// Correction of (b, q-head) gw, the two feature halves' partials summed (written by
// other CTAs of the split grid: read through L2); lane: {C_d, C_n[4 lane .. 4 lane + 3]}
__device__ __forceinline__ void load_corr(const DecArgs& a, size_t gw, int lane, float (&cb)[5]) {
  const float* c0 = a.corr + gw * (1 + D);
  const float* c1 = c0 + a.corr_half;
  const bool two = a.corr_split == 2;
  cb[0] = two ? __ldcg(c0) + __ldcg(c1) : __ldcg(c0);
#pragma unroll
  for (int e = 0; e < 4; ++e)
    cb[1 + e] = two ? __ldcg(c0 + 1 + 4 * lane + e) + __ldcg(c1 + 1 + 4 * lane + e) : __ldcg(c0 + 1 + 4 * lane + e);
}
// partial mode: the summed correction row into the caller's buffer
__device__ __forceinline__ void store_corr_ext(const DecArgs& a, size_t gw, int lane, const float (&cb)[5]) {
  float* o = a.corr_ext + gw * (1 + D);
  if (lane == 0) o[0] = cb[0];
#pragma unroll
  for (int e = 0; e < 4; ++e) o[1 + 4 * lane + e] = cb[1 + e];
}

// LSE merge of one (b, q-head)'s split records (+ the correction) by one warp:
// lanes hold the records' (m, l) for the weights, the numerators stream with
// independent loads; records are read with ld.global.cg (written by other CTAs
// of the same launch).
__device__ __forceinline__ void combine_head(const DecArgs& a, int NG, int b, int h_local, int kvh,
                                             int lane) {
  const int unit = b * a.c.Hkv + kvh, qh = kvh * NG + h_local, gw = b * a.c.Hq + qh;
  const float* base = a.rec + (size_t)unit * a.nrec * NG * REC + (size_t)h_local * REC;
  const size_t rstride = (size_t)NG * REC;
  // record headers (m, l, m_true, -): lane r holds records r, r + 32 (<= 64 records per
  // unit, the planner's cap of 52 plus the residual halves), one load round for the max
  // and the weights
  float4 hd[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int r = 32 * j + lane;
    hd[j] = r < a.nrec ? __ldcg(reinterpret_cast<const float4*>(base + r * rstride))
                       : make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
  }
  float mx = fmaxf(hd[0].x, hd[1].x), mtx = fmaxf(hd[0].z, hd[1].z);
  for (int r = 64 + lane; r < a.nrec; r += 32) {  // longer plans (explicit chunks_per_split)
    const float4 x = __ldcg(reinterpret_cast<const float4*>(base + r * rstride));
    mx = fmaxf(mx, x.x);
    mtx = fmaxf(mtx, x.z);
  }
  float M = warp_max(mx);
  const float Mt = warp_max(mtx);
  float nr[4] = {0.f, 0.f, 0.f, 0.f}, nw[4] = {0.f, 0.f, 0.f, 0.f}, den = 0.f;
  if (M != -INFINITY) {
    for (int r0 = 0; r0 < a.nrec; r0 += 32) {
      const int r = r0 + lane, cnt = min(32, a.nrec - r0);
      float w = 0.f;
      if (r < a.nrec) {
        float m, l;
        if (r0 < 64) {
          m = r0 == 0 ? hd[0].x : hd[1].x;
          l = r0 == 0 ? hd[0].y : hd[1].y;
        } else {
          m = __ldcg(base + r * rstride);
          l = __ldcg(base + r * rstride + 1);
        }
        w = m == -INFINITY ? 0.f : exp2f(m - M);
        den = fmaf(w, l, den);
      }
      // batches of CB records: all CB loads in flight before the accumulation (long-context
      // units have up to 52 + 2 records per head)
#ifndef KVLC_COMBINE_BATCH
#define KVLC_COMBINE_BATCH 8
#endif
      constexpr int CB = KVLC_COMBINE_BATCH;
      for (int i0 = 0; i0 < cnt; i0 += CB) {
        float4 y[CB];
        float wv[CB];
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int i = i0 + u;
          wv[u] = __shfl_sync(0xffffffffu, w, i & 31);
          y[u] = i < cnt ? __ldcg(reinterpret_cast<const float4*>(base + (r0 + i) * rstride + 4) + lane)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < CB; ++u) {
          const int i = i0 + u;
          if (i >= cnt) break;
          float* acc = r0 + i < a.qrec ? nr : nw;  // warp-uniform: quantized (rotated) vs residual (raw) basis
          acc[0] = fmaf(wv[u], y[u].x, acc[0]);
          acc[1] = fmaf(wv[u], y[u].y, acc[1]);
          acc[2] = fmaf(wv[u], y[u].z, acc[2]);
          acc[3] = fmaf(wv[u], y[u].w, acc[3]);
        }
      }
    }
    den = warp_sum(den);
  }
  float cbuf[1 + 4];
  if (a.corr_on) load_corr(a, gw, lane, cbuf);
  if (a.rec_out) {  // partial mode: (M, den, Mt, 0, num_rot, num_raw), correction to corr_ext
    float* o = a.rec_out + (size_t)gw * PREC;
    if (lane == 0) *reinterpret_cast<float4*>(o) = make_float4(M, den, Mt, 0.f);
    *reinterpret_cast<float4*>(o + 4 + 4 * lane) = make_float4(nr[0], nr[1], nr[2], nr[3]);
    *reinterpret_cast<float4*>(o + 4 + D + 4 * lane) = make_float4(nw[0], nw[1], nw[2], nw[3]);
    if (a.corr_on && a.corr_ext) store_corr_ext(a, gw, lane, cbuf);
    return;
  }
  void* o = a.out_fp32 ? (void*)(static_cast<float*>(a.out) + (size_t)gw * D)
                       : (void*)(static_cast<uint16_t*>(a.out) + (size_t)gw * D);
  finish(M, Mt, den, nr, nw, a.corr_on ? cbuf : nullptr, a.literal, lane, o, a.out_fp32);
}

// The whole decode step's split-KV work in one launch; blockIdx selects the
// task: quantized splits, residual halves, correction rows.  Every CTA bumps
// its unit's arrival counter after publishing its record; the last one
// performs the LSE combine of the unit (no separate combine launch).

#ifndef KVLC_SPLIT_MINB
#define KVLC_SPLIT_MINB 4
#endif
// WPC: quantized splits run warp per chunk (kvlc_quant_wpc.cuh, dynamic shared memory)
// instead of warp per 32-token slice (kvlc_quant.cuh, static shared memory)
// One task of the split grid: correction rows, a quantized split or a residual half.
template <int NG, int EXTRA, bool WPC>
__device__ __forceinline__ int run_task(const DecArgs& a, unsigned char* smem, int x) {
  SplitSmem& sm = *reinterpret_cast<SplitSmem*>(smem);
  float* const smrec = reinterpret_cast<float*>(smem);
  const int U = a.c.B * a.c.Hkv;
  const int ncorr = a.tail && a.corr_on ? a.corr_split * U : 0;  // correction tasks first (S overlaps codes)
  int unit;
  if (x < ncorr) {
    unit = a.corr_split == 2 ? x >> 1 : x;
#ifndef KVLC_PROBE_NOCORR  // probe build: correction CTAs exit at once (timing only)
    if (a.corr_split == 2)
      run_corr<NG>(a, unit, x & 1, smrec);
    else
      run_corr_unit<NG>(a, unit, smrec);
#endif
    if (a.tail_fused) {  // the residual half h of the same unit (tail tasks: one start-up)
      __syncthreads();
      run_resid<NG>(a, unit, x & 1, smrec);
    }
  } else if ((x -= ncorr) < U * a.nsq) {
    unit = x / a.nsq;
    if (WPC)
      run_quant_wpc<NG, EXTRA>(a, unit, x % a.nsq, *reinterpret_cast<WpcSmem*>(smem), smrec);
    else
      run_quant<NG, EXTRA>(a, unit, x % a.nsq, sm);
  } else {
    x -= U * a.nsq;
    unit = x / 2;
    run_resid<NG>(a, unit, x % 2, smrec);
  }
  return unit;
}

template <int NG, int EXTRA, bool WPC>
__device__ __forceinline__ void split_body(const DecArgs& a, unsigned char* smem) {
  __shared__ int last;
  __shared__ int next;
  int x = blockIdx.x, unit;
#ifdef KVLC_TRACE
  const unsigned long long t_enter = gtimer();
#endif
  // One call site of run_task (inlined): with a task counter (persistent warp-per-chunk
  // grid) the CTA runs task blockIdx.x first (its code stream may start before the
  // predecessor grid completes), then tasks gridDim.x + (ticket of the counter) in order,
  // so CTAs that finish early take the remaining splits and residual halves and no slot
  // idles while another wave waits.  The last ticket resets the counter.
  for (;;) {
    unit = run_task<NG, EXTRA, WPC>(a, smem, x);
    if (!WPC || a.queue == nullptr) break;
    __syncthreads();  // every warp is done with the task's shared memory
    if (threadIdx.x == 0) {
      const uint32_t d = atomicAdd(a.queue, 1u);
      if (d == (uint32_t)(a.ntask - 1)) *a.queue = 0u;
      next = (int)d + gridDim.x;
    }
    __syncthreads();
    x = next;
    if (x >= a.ntask) break;
  }
#ifdef KVLC_TRACE
  __syncthreads();
  DT_STAMP(0, t_enter);
  DT_STAMP(1, gtimer());
  {
    const int U = a.c.B * a.c.Hkv, ncorr = a.tail && a.corr_on ? a.corr_split * U : 0;
    DT_STAMP(3, ((unsigned long long)smid() << 32) |
                    (unsigned long long)((blockIdx.x < ncorr ? 0 : blockIdx.x < ncorr + U * a.nsq ? 1 : 2) << 24 | unit));
  }
  if (a.sep_combine) DT_STAMP(2, gtimer());
#endif
  if (a.sep_combine) {
    griddep_launch();  // the combine kernel may be scheduled; it waits for this grid to complete
    return;
  }
  const int per_unit = a.nsq + (a.tail ? (a.tail_fused ? 0 : 2) + (a.corr_on ? a.corr_split : 0) : 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    griddep_wait();   // the predecessor grid (if any) has flushed: counters / q are current
    __threadfence();  // publish this CTA's record / correction rows
    last = atomicAdd(a.done + unit, 1u) == (uint32_t)(per_unit - 1);
  }
  __syncthreads();
  if (!last) {
    DT_STAMP(2, gtimer());
    return;
  }
  __threadfence();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = unit / a.c.Hkv, kvh = unit % a.c.Hkv;
  for (int h = warp; h < NG; h += WARPS) combine_head(a, NG, b, h, kvh, lane);
  if (threadIdx.x == 0) a.done[unit] = 0u;  // self-cleaning for the next step
#ifdef KVLC_TRACE
  __syncthreads();
  DT_STAMP(2, gtimer() | (1ull << 63));  // top bit: this CTA ran the unit's combine
#endif
}

template <int NG, int EXTRA>
__global__ void __launch_bounds__(THREADS, KVLC_SPLIT_MINB) split_kernel(const DecArgs a) {
  __shared__ __align__(16) SplitSmem sm;
  split_body<NG, EXTRA, false>(a, reinterpret_cast<unsigned char*>(&sm));
}

// 55 KB of dynamic shared memory per CTA: 4 CTAs per SM for groups of <= 4 heads (q in
// shared memory, 128 registers), 3 for larger groups (q and the lo B parts in registers)
// CTAs per SM of the warp-per-chunk kernel for groups of <= 4 heads: 3 (162 registers) measured
// faster than 4 (the 128-register cap) and 2: config 2 kernel pair 36.4 -> 34.7 us (2: 42.3),
// config 4 28.9 -> 28.6, config 1 8.6 -> 8.4 (tools/run_abvar.sh, r02)
#ifndef KVLC_WPC_MINB4
#define KVLC_WPC_MINB4 3
#endif
#ifndef KVLC_WPC_MINB8
#define KVLC_WPC_MINB8 3  // the same for groups of 5-8 heads
#endif
constexpr int wpc_minb(int ng) { return ng <= 4 ? KVLC_WPC_MINB4 : KVLC_WPC_MINB8; }
template <int NG, int EXTRA>
__global__ void __launch_bounds__(THREADS, wpc_minb(NG)) split_kernel_wpc(const DecArgs a) {
  extern __shared__ __align__(128) unsigned char dsm[];
  split_body<NG, EXTRA, true>(a, dsm);
}

// The LSE combine as its own launch (programmatic dependent of split_kernel), used when a
// unit has at most CMB_MAXREC records: one CTA per (b, q-head), warp w takes records
// w, w + 4, ..., lane l channels 4l .. 4l+3.  Every load (record numerators, headers,
// correction row) is issued in one round after the split grid has completed; the
// 4 warps' partial sums meet in shared memory and warp 0 applies the correction,
// the FWHT and the divide (finish).
constexpr int CMB_PER_WARP = 16;                  // numerators held in registers per lane
constexpr int CMB_MAXREC = WARPS * CMB_PER_WARP;  // 64

template <int NG>
__global__ void __launch_bounds__(THREADS) combine_kernel(const DecArgs a) {
  __shared__ float hm[CMB_MAXREC];   // record weights
  __shared__ float red[3][WARPS];    // max m, max m_true, den
  __shared__ __align__(16) float part[WARPS - 1][2][D];
  const int gw = blockIdx.x, b = gw / a.c.Hq, qh = gw % a.c.Hq, kvh = qh / NG, hl = qh % NG;
  const int unit = b * a.c.Hkv + kvh;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const float* base = a.rec + ((size_t)unit * a.nrec * NG + hl) * REC;
  const size_t rs = (size_t)NG * REC;
  const int nrec = a.nrec;
  griddep_wait();
  float4 y[CMB_PER_WARP];
#pragma unroll
  for (int i = 0; i < CMB_PER_WARP; ++i) {
    const int r = warp + WARPS * i;
    y[i] = r < nrec ? __ldcg(reinterpret_cast<const float4*>(base + r * rs + 4) + lane)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float4 hd = t < nrec ? __ldcg(reinterpret_cast<const float4*>(base + t * rs))
                             : make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
  float cbuf[1 + 4];
  if (a.corr_on && warp == 0) load_corr(a, gw, lane, cbuf);
  float m = warp_max(hd.x), mt = warp_max(hd.z);
  if (lane == 0) {
    red[0][warp] = m;
    red[1][warp] = mt;
  }
  __syncthreads();
  float M = red[0][0], Mt = red[1][0];
#pragma unroll
  for (int w = 1; w < WARPS; ++w) {
    M = fmaxf(M, red[0][w]);
    Mt = fmaxf(Mt, red[1][w]);
  }
  const float wt = hd.x == -INFINITY ? 0.f : exp2f(hd.x - M);
  if (t < nrec) hm[t] = wt;
  const float dsum = warp_sum(wt * hd.y);
  if (lane == 0) red[2][warp] = dsum;
  __syncthreads();
  float nr[4] = {0.f, 0.f, 0.f, 0.f}, nw[4] = {0.f, 0.f, 0.f, 0.f};
  if (M != -INFINITY) {
#pragma unroll
    for (int i = 0; i < CMB_PER_WARP; ++i) {
      const int r = warp + WARPS * i;
      if (r >= nrec) break;
      const float w = hm[r];
      float* acc = r < a.qrec ? nr : nw;  // quantized (rotated) vs residual (raw) basis
      acc[0] = fmaf(w, y[i].x, acc[0]);
      acc[1] = fmaf(w, y[i].y, acc[1]);
      acc[2] = fmaf(w, y[i].z, acc[2]);
      acc[3] = fmaf(w, y[i].w, acc[3]);
    }
  }
  if (warp > 0) {
    *reinterpret_cast<float4*>(&part[warp - 1][0][4 * lane]) = make_float4(nr[0], nr[1], nr[2], nr[3]);
    *reinterpret_cast<float4*>(&part[warp - 1][1][4 * lane]) = make_float4(nw[0], nw[1], nw[2], nw[3]);
  }
  __syncthreads();
  if (warp > 0) return;
  float den = 0.f;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) den += red[2][w];
#pragma unroll
  for (int w = 0; w < WARPS - 1; ++w) {
    const float4 x = *reinterpret_cast<const float4*>(&part[w][0][4 * lane]);
    const float4 z = *reinterpret_cast<const float4*>(&part[w][1][4 * lane]);
    nr[0] += x.x; nr[1] += x.y; nr[2] += x.z; nr[3] += x.w;
    nw[0] += z.x; nw[1] += z.y; nw[2] += z.z; nw[3] += z.w;
  }
  if (M == -INFINITY) den = 0.f;
  if (a.rec_out) {  // partial mode: (M, den, Mt, 0, num_rot, num_raw), correction to corr_ext
    float* o = a.rec_out + (size_t)gw * PREC;
    if (lane == 0) *reinterpret_cast<float4*>(o) = make_float4(M, den, Mt, 0.f);
    *reinterpret_cast<float4*>(o + 4 + 4 * lane) = make_float4(nr[0], nr[1], nr[2], nr[3]);
    *reinterpret_cast<float4*>(o + 4 + D + 4 * lane) = make_float4(nw[0], nw[1], nw[2], nw[3]);
    if (a.corr_on && a.corr_ext) store_corr_ext(a, gw, lane, cbuf);
    return;
  }
  void* o = a.out_fp32 ? (void*)(static_cast<float*>(a.out) + (size_t)gw * D)
                       : (void*)(static_cast<uint16_t*>(a.out) + (size_t)gw * D);
  finish(M, Mt, den, nr, nw, a.corr_on ? cbuf : nullptr, a.literal, lane, o, a.out_fp32);
}

// Copies a step's input (q) from pinned host memory to the device with every 16-byte
// piece in flight at once, and lets the programmatic-launch dependent (the decode)
// start its code streams immediately: inside a CUDA graph a copy-engine H2D node
// followed by the kernel costs ~18 us per step, this pair ~4 us (tools/bench_e2e.py).
__global__ void __launch_bounds__(256) stage_input_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                          size_t n16) {
  griddep_launch();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// LSE merge of n device records (m, l, y_rot, y_raw) + correction -> out.
__global__ void __launch_bounds__(128) merge_records_kernel(const float* __restrict__ recs, int n,
                                                            int64_t stride, const float* __restrict__ corr,
                                                            int BH, int literal, int out_fp32,
                                                            void* __restrict__ out) {
  const int gw = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gw >= BH) return;
  float M = -INFINITY, Mt = -INFINITY;
  for (int r = 0; r < n; ++r) {
    M = fmaxf(M, recs[r * stride + (size_t)gw * PREC]);
    Mt = fmaxf(Mt, recs[r * stride + (size_t)gw * PREC + 2]);
  }
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
  float cbuf[5];
  if (corr) {
    const float* cp = corr + (size_t)gw * (1 + D);
    cbuf[0] = cp[0];
#pragma unroll
    for (int e = 0; e < 4; ++e) cbuf[1 + e] = cp[1 + 4 * lane + e];
  }
  finish(M, Mt, den, nr, nw, corr ? cbuf : nullptr, literal, lane, o, out_fp32);
}

// Per-block partials of decode_step_blocked (return_partials, attention.py:41-47, 269-275) from
// the records of a decode whose splits are the blocks (cpc chunks each): block i < ceil(n_chunks /
// cpc) (the quantized blocks of cpc G tokens, stored basis; a split's rps warp records merged) and
// one residual block (the two ring halves merged), converted from the kernel's log2-unit
// reference points to the reference's natural-unit block max: m = m_true ln 2, l and y scaled
// by 2^(m_ref - m_true).  out: [B][Hq][max_blocks][2 + D].
__global__ void __launch_bounds__(128) blocks_kernel(const kvlc_cache c, const float* __restrict__ rec, int nrec,
                                                     int nsq, int rps, int cpc, int NG, int max_blocks,
                                                     float* __restrict__ out) {
  const int gw = blockIdx.x, b = gw / c.Hq, qh = gw % c.Hq, kvh = qh / NG, hl = qh % NG;
  const int unit = b * c.Hkv + kvh;
  const int nq = min((c.n_chunks[b] + cpc - 1) / cpc, nsq), has_res = c.res_len[b] > 0 ? 1 : 0;
  const size_t rs = (size_t)NG * REC;
  const float* base = rec + ((size_t)unit * nrec * NG + hl) * REC;
  float* o = out + (size_t)gw * max_blocks * (2 + D);
  const float LN2 = 0.6931471805599453f;
  for (int i = 0; i < max_blocks; ++i) {
    float m = 0.f, l = 0.f, f0 = 0.f, f1 = 0.f;
    const float *y0 = nullptr, *y1 = nullptr;
    if (i < nq && rps > 1) {  // a block of several warp records: merged at the block's true max
      const float* r = base + (size_t)i * rps * rs;
      float M = -INFINITY;
      for (int w = 0; w < rps; ++w) M = fmaxf(M, r[w * rs + 2]);
      float y = 0.f;
      for (int w = 0; w < rps; ++w) {
        const float* rw = r + w * rs;
        const float f = rw[0] == -INFINITY ? 0.f : exp2f(rw[0] - M);
        l = fmaf(rw[1], f, l);
        y = fmaf(rw[4 + threadIdx.x], f, y);
      }
      if (threadIdx.x == 0) {
        o[i * (2 + D)] = M * LN2;
        o[i * (2 + D) + 1] = l;
      }
      o[i * (2 + D) + 2 + threadIdx.x] = y;
      continue;
    }
    if (i < nq) {
      const float* r = base + (size_t)i * rps * rs;  // one record per block
      f0 = r[2] == -INFINITY ? 0.f : exp2f(r[0] - r[2]);
      m = r[2] * LN2;
      l = r[1] * f0;
      y0 = r + 4;
    } else if (i == nq && has_res) {
      const float* r0 = base + (size_t)nsq * rps * rs;
      const float* r1 = r0 + rs;
      const float M = fmaxf(r0[2], r1[2]);
      f0 = r0[0] == -INFINITY ? 0.f : exp2f(r0[0] - M);
      f1 = r1[0] == -INFINITY ? 0.f : exp2f(r1[0] - M);
      m = M * LN2;
      l = r0[1] * f0 + r1[1] * f1;
      y0 = r0 + 4;
      y1 = r1 + 4;
    }
    if (threadIdx.x == 0) {
      o[i * (2 + D)] = m;
      o[i * (2 + D) + 1] = l;
    }
    const int ch = threadIdx.x;
    float y = 0.f;
    if (y0) y = y0[ch] * f0;
    if (y1) y = fmaf(y1[ch], f1, y);
    o[i * (2 + D) + 2 + ch] = y;
  }
}

// ------------------------------------------------------------- host ----
// Quantized splits warp per chunk or warp per 32-token slice.  Same-box A/B (r02,
// tools/run_var.sh): config 2 (4 heads per group) 37.0 vs 36.8 us, config 4 29.7 vs 33.5 us,
// config 3 (7 heads: 150+ registers, 3 CTAs per SM) 26.9-28.8 vs 24.9 us; so warp per chunk
// for groups of <= 4 heads.  KVLC_WPC=0 / 1 forces either (A/B).
// Warp-per-chunk splits for a group of ng heads over `span` chunks per unit.  Groups of <= 4
// heads always; larger groups (config 3's 7) from ~100 chunks: B16 x 16k 46.1 -> 44.7 us,
// B64 x 16k 148.6 -> 143.8, B16 x 32k 76.8 -> 72.6, B64 x 32k 265.6 -> 243.4; shorter
// contexts lose (B16 x 8k 26.7 -> 31.8, B16 x 4k 21.5 -> 22.5).  KVLC_WPC=0/1 forces.
bool wpc_for(int ng, int span) {
  static const int v = [] {
    const char* e = getenv("KVLC_WPC");
    return e ? atoi(e) : -1;
  }();
  return v < 0 ? (ng <= 4 || span >= 100) : v != 0;
}
int split_minb(int ng, bool wpc) { return wpc ? wpc_minb(ng) : KVLC_SPLIT_MINB; }

struct Plan {
  int NG, U, nsq, cpc, nrec, corr_on, rps, qrec, wpc;
  size_t done_off, corr_off, rec_off, total;
};

int plan_for(const kvlc_cache* c, const kvlc_decode_opts* o, int chunk_lo, int chunk_hi, int tail,
             bool corr_on, Plan& p) {
  KVLC_REQUIRE(c && c->B >= 1 && c->Hkv >= 1 && c->Hq % c->Hkv == 0 && c->Hq / c->Hkv <= 8,
               "bad cache dims");
  p.NG = c->Hq / c->Hkv;
  p.U = c->B * c->Hkv;
  int maxc = o && o->max_chunks_hint > 0 ? o->max_chunks_hint : c->max_chunks;
  int span = std::max(0, std::min(maxc, chunk_hi) - chunk_lo);
  static const int cpc_env = [] {  // tuning override (tools/run_dec.sh sweeps)
    const char* e = getenv("KVLC_CPC");
    return e ? atoi(e) : 0;
  }();
  int cpc = o && o->chunks_per_split > 0 ? o->chunks_per_split : cpc_env;
  p.wpc = wpc_for(p.NG, span) ? 1 : 0;
  if (cpc == 0 && p.wpc) {
    // warp per chunk: a split's 4 warps take every 4th chunk, so splits are sized in
    // whole chunks per warp (balanced warps; the CTA waits for its slowest warp before
    // merging).  About one wave of splits at WPC_MINB CTAs per SM, at most 52 records per
    // unit, then equal splits rounded up to a multiple of 4 chunks.
    const long long warps = 148LL * wpc_minb(p.NG) * WARPS;
    const long long chunks = (long long)p.U * std::max(span, 1);
    // chunks per warp; multi-wave workloads keep splits short (the tail of the last wave)
    // at most 6 chunks per warp, 4 for groups above 4 heads (their chunk costs more: Qwen B16 x 32k
    // 72.2 -> 67.1 us; Llama B64 x 8k prefers 6: 115.3 vs 117.9).  KVLC_CPWCAP overrides (A/B)
    static const int cpw_env = [] {
      const char* e = getenv("KVLC_CPWCAP");
      return e ? atoi(e) : 0;
    }();
    const long long cpw_cap = cpw_env ? cpw_env : (p.NG > 4 ? 4 : 6);
    long long cpw = std::min(cpw_cap, std::max(2LL, (chunks + warps / 2) / warps));
    long long nsq = (std::max(span, 1) + 4 * cpw - 1) / (4 * cpw);
    static const int rec_cap = [] {
      const char* e = getenv("KVLC_RECCAP");
      return e ? atoi(e) : 52;
    }();
    nsq = std::max(1LL, std::min(nsq, (long long)rec_cap));
    long long per = (std::max(span, 1) + nsq - 1) / nsq;
    per = (per + 3) / 4 * 4;
    cpc = (int)std::max(4LL, std::min(128LL, per));
  } else if (cpc == 0) {
    // Per-CTA fixed cost (pipeline fill, q / B build, record merge, arrival) favours
    // long splits; the tail favours many.  Measured on configs 2-4
    // (tools/run_cpc3.sh, run_cpc4.sh): about 1.5 waves of splits at
    // KVLC_SPLIT_MINB CTAs per SM, at least 8 chunks per split, at most 52 records per
    // unit (the last CTA of a unit merges them all), then equal-length splits.
    // Configs 2 / 3 / 4: 7 -> 9 / 8 / 20 chunks, 49.2 -> 44.4 / 38.1 -> 34.8 / 55.6 -> 46.5 us.
    // Rounded (not ceiled) wave target: 64 chunks per unit get 8 x 8 rather than 6 x 10 + 4.
    const long long slots = 148LL * split_minb(p.NG, p.wpc);
    const long long chunks = (long long)p.U * std::max(span, 1);
    long long t = std::max(8LL, (4 * chunks + 3 * slots) / (6 * slots));  // round(chunks / (1.5 slots))
    static const int rec_cap = [] {
      const char* e = getenv("KVLC_RECCAP");
      return e ? atoi(e) : 52;
    }();
    t = std::max(t, (long long)(std::max(span, 1) + rec_cap - 1) / rec_cap);
    const long long nsq = (std::max(span, 1) + t - 1) / t;
    cpc = (int)std::max(1LL, std::min(32LL, (std::max(span, 1) + nsq - 1) / nsq));
  }
  p.cpc = cpc;
  p.nsq = std::max(1, (span + cpc - 1) / cpc);
  p.corr_on = corr_on && tail ? 1 : 0;
  // warp-per-chunk splits write one record per warp (no CTA merge) while the combine can
  // hold them all (KVLC_WARPREC=0: CTA-merged records, A/B)
  static const int warprec_env = [] {
    const char* e = getenv("KVLC_WARPREC");
    return e ? atoi(e) : 1;
  }();
  p.rps = (warprec_env && p.wpc && 4 * p.nsq + (tail ? 2 : 0) <= 64) ? 4 : 1;
  p.qrec = p.nsq * p.rps;
  p.nrec = p.qrec + (tail ? 2 : 0);
  size_t BH = (size_t)c->B * c->Hq;
  p.corr_off = 0;
  p.rec_off = align_up(2 * BH * (1 + D) * sizeof(float));  // correction partials of the 2 halves
  // arrival counters first: their offset must not depend on the split plan
  // (they are zero-initialised once and left at zero by every launch)
  p.done_off = 0;
  const size_t base = align_up((size_t)(p.U + 1) * sizeof(uint32_t));  // + the task counter
  p.corr_off += base;
  p.rec_off += base;
  p.total = p.rec_off + align_up((size_t)p.U * p.nrec * p.NG * REC * sizeof(float));
  return KVLC_OK;
}

template <int NG>
int launch_ng(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q, const Plan& p,
              char* ws, int chunk_lo, int chunk_hi, int tail, float* corr_ext, int literal,
              int out_fp32, void* out, float* rec_out, const kvlc_decode_opts* o, cudaStream_t s) {
  float* corr = reinterpret_cast<float*>(ws + p.corr_off);  // the halves; the combine sums them
  float* rec = reinterpret_cast<float*>(ws + p.rec_off);
  DecArgs a{};
  a.c = *c;
  a.q = q;
  if (p.corr_on) {
    a.w1q = ad->w1q;
    a.w2q = ad->w2q;
  }
  a.corr = corr;
  a.corr_half = (size_t)c->B * c->Hq * (1 + D);
  a.corr_ext = corr_ext;
  a.rec = rec;
  a.nsq = p.nsq;
  a.rps = p.rps;
  a.qrec = p.qrec;
  a.cpc = p.cpc;
  a.chunk_lo = chunk_lo;
  a.chunk_hi = chunk_hi;
  a.tail = tail;
  a.corr_on = p.corr_on;
  a.nrec = p.nrec;
  a.done = reinterpret_cast<uint32_t*>(ws + p.done_off);
  a.literal = literal;
  a.out_fp32 = out_fp32;
  a.out = out;
  a.rec_out = rec_out;
  // combine placement: its own PDL-chained kernel (config 2 / 3 / 4: 42.7 -> 40.1,
  // 32.4 -> 27.4, 41.4 -> 35.1 us: the split CTAs skip the fence + arrival atomic, ~1.2 us
  // each, and the combine is one load round per head, tools/trace_decode.py), or the last
  // arriving CTA of each unit for plans with more records than combine_kernel holds
  static const int sep_env = [] {  // KVLC_SEPCOMB=0 forces the fused combine (A/B)
    const char* e = getenv("KVLC_SEPCOMB");
    return e ? atoi(e) : 1;
  }();
  a.sep_combine = sep_env && p.nrec <= CMB_MAXREC;
  // correction halves (two CTAs per unit) shorten the grid's longest task; they pay only
  // when the splits spill past one wave anyway (config 2: 38.0 -> 37.3 us; config 3, whose
  // splits + whole-unit corrections fit one wave: 26.6 -> 30.9 us with halves)
  static const int corr_split_env = [] {  // KVLC_CORRSPLIT=1/2 forces (A/B)
    const char* e = getenv("KVLC_CORRSPLIT");
    return e ? atoi(e) : 0;
  }();
  // r02 late (3 warp-per-chunk CTAs per SM): groups of <= 4 heads take the halves in every grid,
  // one wave included (B1 x 4k, 8 kv heads x 4 heads: 10.70 -> 8.48 us; B1 x 1k x 8 MHA heads
  // 8.25 -> 7.72; B4 x 4k 13.97 -> 11.67; B1 x 32k 14.62 -> 13.29)
  a.corr_split = corr_split_env ? corr_split_env
                                : ((NG <= 4 || (long long)p.U * (p.nsq + 1) > 148LL * split_minb(NG, p.wpc)) ? 2 : 1);
  // tail tasks: correction half h + residual half h in one CTA (one start-up and q staging
  // instead of two; both are latency-bound) when the correction runs in halves
  static const int tailfuse_env = [] {
    const char* e = getenv("KVLC_TAILFUSE");
    return e ? atoi(e) : 1;
  }();
  // Measured (r02, same box): one-wave grids gain (config 3 B1 x 4k 16.0 -> 13.3 us, B16 x 4k
  // 24.9 -> 21.3), multi-wave grids lose (config 2 36.8 -> 38.6, config 3 B16 x 8k 26.4 -> 31.0:
  // the long tail tasks hold slots the splits need), so fused only when everything fits one wave.
  // And only for groups of more than 4 heads: after the correction unit's phi loads were
  // batched, one-wave grids of small groups run faster with a whole-unit correction CTA beside
  // two residual CTAs (B1 x 4k, 8 kv heads: NG 1 9.29 -> 8.59 us, NG 2 9.43 -> 9.26, NG 4
  // 10.29 -> 10.49, NG 4 at 32k 15.55 -> 14.65, NG 8 13.36 -> 16.43; Qwen NG 7 keeps fusing:
  // B1 x 32k 13.9 vs 15.3).  KVLC_TAILFUSE=0 off, 1 auto, 2 any group size.
  const bool one_wave = (long long)p.U * (p.nsq + 2) <= 148LL * split_minb(NG, p.wpc);
  const bool fuse = tailfuse_env == 2 || (tailfuse_env == 1 && NG > 4);
  if (tail && p.corr_on && fuse && one_wave && !corr_split_env) a.corr_split = 2;
  a.tail_fused = tail && p.corr_on && a.corr_split == 2 && fuse && one_wave;
  int grid = p.U * p.nsq + (tail ? (a.tail_fused ? 0 : 2 * p.U) + (p.corr_on ? a.corr_split * p.U : 0) : 0);
  // persistent split grid (warp-per-chunk kernel, separate combine): at most one wave of
  // CTAs that take tasks from a counter.  Measured slower (config 2 split 37.0 -> 38.1 us
  // same box, r02: every task keeps its start-up and record costs, and late long tasks
  // stretch the tail), so off unless KVLC_DYN=1.
  static const int dyn_env = [] {
    const char* e = getenv("KVLC_DYN");
    return e ? atoi(e) : 0;
  }();
  a.ntask = grid;
  a.queue = nullptr;
  if (p.wpc && a.sep_combine && dyn_env) {
    a.queue = reinterpret_cast<uint32_t*>(ws + p.done_off) + p.U;
    grid = std::min(grid, 148 * split_minb(NG, true));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.stream = s;
  // programmatic dependent launch: CTAs may start while the predecessor kernel (the
  // previous step's combine, or kvlc_stage_input's copy of q) finishes; every read of q or
  // of the arrival counters follows griddepcontrol.wait, the code streams do not, so after
  // an entry point that wrote cache state (prefill / append / flush / deserialize) the
  // launch waits fully (take_cache_write)
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = take_cache_write(c) ? 0 : 1;  // the cache was written since its last decode: full wait
  if (o && o->ev_begin) KVLC_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(o->ev_begin), s));
  // precision passes for > 4 heads per group (see quant_chunk); KVLC_EXTRA overrides (tuning)
  static const int extra_env = [] {
    const char* e = getenv("KVLC_EXTRA");
    return e ? atoi(e) & 3 : 3;
  }();
  const int extra = NG <= 4 ? 0 : extra_env;
  if (p.wpc) {
    static bool attr_set[4] = {false, false, false, false};
    void (*kfn)(const DecArgs) = NG <= 4 || extra == 0 ? split_kernel_wpc<NG, 0>
                                 : extra == 1            ? split_kernel_wpc<NG, NG <= 4 ? 0 : 1>
                                 : extra == 2            ? split_kernel_wpc<NG, NG <= 4 ? 0 : 2>
                                                         : split_kernel_wpc<NG, NG <= 4 ? 0 : 3>;
    if (!attr_set[extra]) {
      KVLC_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WPC_SMEM));
      attr_set[extra] = true;
    }
    cfg.dynamicSmemBytes = WPC_SMEM;
    KVLC_CUDA(cudaLaunchKernelEx(&cfg, kfn, a));
    cfg.dynamicSmemBytes = 0;
  } else {
    void (*kfn)(const DecArgs) = NG <= 4 || extra == 0 ? split_kernel<NG, 0>
                                 : extra == 1            ? split_kernel<NG, NG <= 4 ? 0 : 1>
                                 : extra == 2            ? split_kernel<NG, NG <= 4 ? 0 : 2>
                                                         : split_kernel<NG, NG <= 4 ? 0 : 3>;
    KVLC_CUDA(cudaLaunchKernelEx(&cfg, kfn, a));
  }
  if (a.sep_combine) {
    cfg.gridDim = dim3(c->B * c->Hq);
    KVLC_CUDA(cudaLaunchKernelEx(&cfg, combine_kernel<NG>, a));
  }
  if (o && o->ev_end) KVLC_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(o->ev_end), s));
  return check_launch("decode");
}

int launch(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q, const Plan& p, char* ws,
           int chunk_lo, int chunk_hi, int tail, float* corr_ext, int literal, int out_fp32, void* out,
           float* rec_out, const kvlc_decode_opts* o, cudaStream_t s) {
  switch (p.NG) {
#define KVLC_NG_CASE(n) \
  case n:               \
    return launch_ng<n>(c, ad, q, p, ws, chunk_lo, chunk_hi, tail, corr_ext, literal, out_fp32, out, rec_out, o, s);
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

#ifdef KVLC_TRACE
extern "C" int kvlc_dphase_copy(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_dphase, bytes < sizeof(g_dphase) ? bytes : sizeof(g_dphase)) == cudaSuccess ? 0 : 2;
}
extern "C" int kvlc_dtrace_copy(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_dtrace, bytes < sizeof(g_dtrace) ? bytes : sizeof(g_dtrace)) == cudaSuccess ? 0 : 2;
}
#endif

extern "C" {

size_t kvlc_decode_workspace(const kvlc_cache* c, const kvlc_decode_opts* o) {
  Plan p{};
  if (!c || plan_for(c, o, 0, 1 << 30, 1, true, p)) return 0;
  return p.total;
}

int kvlc_decode(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q, void* out,
                const kvlc_decode_opts* o, void* ws, size_t ws_bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(q && out, "null query / output");
  Plan p{};
  int rc = plan_for(c, o, 0, 1 << 30, 1, adapter_active(ad), p);
  if (rc) return rc;
  KVLC_REQUIRE(ws && ws_bytes >= p.total, "decode workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
  return launch(c, ad, q, p, static_cast<char*>(ws), 0, 1 << 30, 1, nullptr, o ? o->literal : 0,
                o ? o->out_fp32 : 0, out, nullptr, o, as_stream(stream));
}

int kvlc_decode_blocks(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q, void* out, float* blocks,
                       int32_t max_blocks, const kvlc_decode_opts* o, void* ws, size_t ws_bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(q && out && blocks, "null query / output / blocks");
  kvlc_decode_opts o1{};
  if (o) o1 = *o;
  // a split per block: block_tokens = chunks_per_split x G (default one chunk)
  if (o1.chunks_per_split <= 0) o1.chunks_per_split = 1;
  Plan p{};
  int rc = plan_for(c, &o1, 0, 1 << 30, 1, adapter_active(ad), p);
  if (rc) return rc;
  KVLC_REQUIRE(ws && ws_bytes >= p.total, "decode workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
  KVLC_REQUIRE(max_blocks >= p.nsq + 1, "blocks buffer holds %d blocks per head, the cache needs %d", max_blocks,
               p.nsq + 1);
  rc = launch(c, ad, q, p, static_cast<char*>(ws), 0, 1 << 30, 1, nullptr, o1.literal, o1.out_fp32, out, nullptr, &o1,
              as_stream(stream));
  if (rc) return rc;
  blocks_kernel<<<c->B * c->Hq, 128, 0, as_stream(stream)>>>(
      *c, reinterpret_cast<const float*>(static_cast<char*>(ws) + p.rec_off), p.nrec, p.nsq, p.rps, p.cpc, p.NG,
      max_blocks, blocks);
  return check_launch("decode_blocks");
}

int kvlc_decode_partial(const kvlc_cache* c, const kvlc_adapter* ad, const uint16_t* q,
                        int32_t chunk_lo, int32_t chunk_hi, int32_t include_tail, float* rec,
                        float* corr, const kvlc_decode_opts* o, void* ws, size_t ws_bytes,
                        void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(q && rec, "null query / record buffer");
  KVLC_REQUIRE(chunk_lo >= 0 && chunk_hi >= chunk_lo, "bad chunk window [%d, %d)", chunk_lo, chunk_hi);
  KVLC_REQUIRE(!include_tail || !adapter_active(ad) || corr, "tail owner needs a correction buffer");
  Plan p{};
  int rc = plan_for(c, o, chunk_lo, chunk_hi, include_tail ? 1 : 0, adapter_active(ad), p);
  if (rc) return rc;
  KVLC_REQUIRE(ws && ws_bytes >= p.total, "decode workspace too small: need %zu bytes, got %zu", p.total, ws_bytes);
  if (include_tail && corr && !p.corr_on)
    KVLC_CUDA(cudaMemsetAsync(corr, 0, (size_t)c->B * c->Hq * (1 + D) * sizeof(float), as_stream(stream)));
  return launch(c, ad, q, p, static_cast<char*>(ws), chunk_lo, chunk_hi, include_tail ? 1 : 0, corr,
                0, 0, nullptr, rec, o, as_stream(stream));
}

int kvlc_stage_input(const void* src, void* dst, size_t bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(src && dst && bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0,
               "stage_input needs 16-byte aligned buffers and a multiple of 16 bytes (%zu)", bytes);
  if (bytes == 0) return KVLC_OK;
  const size_t n16 = bytes / 16;
  const int grid = (int)std::min<size_t>((n16 + 255) / 256, 148 * 8);
  stage_input_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst),
                                                          n16);
  return check_launch("stage_input");
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
