// Quantized-split path of the fused decode (included by kvlc_decode.cu).
//
// A quantized-split CTA owns chunks [lo, hi) of one (b, kv-head) unit.  Its
// 4 warps take the 4 32-token slices of every chunk:
//   * thread 0 streams whole chunks (4 KB K codes, 4 KB V codes, 4 x 256 B
//     scales / zeros, the bytes of the global layouts) into a STAGES-deep ring
//     of shared-memory stages with bulk copies (TMA, one transaction-count
//     mbarrier per stage; 4 warp arrivals free a stage): up to STAGES - 1 chunks
//     in flight per CTA without LSU request tracking (per-warp 16-B cp.async
//     streaming topped out near 3.3 TB/s with the math removed);
//   * the QK^T B operand of a chunk (q' = q * s_k, fp16 hi/lo) and the zero
//     term zt = q . z_k are built cooperatively (warp w: k-tiles 2w, 2w+1) into
//     shared buffers guarded by full / empty mbarriers (4 warp arrivals each):
//     a warp waits only for the B shares it is about to read, not at a CTA
//     barrier per chunk (43.7 vs 45.1 us on config 2);
//   * codes become fp16 MMA operands with one LOP3 per register (exact
//     subnormals c * 4^j * 2^-24 from the fragment-native layouts written by
//     kvlc_flush.cu); mma.sync m16n8k16, GQA heads on N;
//   * online softmax in log2 units with lazy rescaling: the reference point
//     only moves when the running max grows by more than LAZY (p <= 2^LAZY),
//     the true max is tracked separately for literal-correction parity.
#pragma once

#ifndef KVLC_STAGES
#define KVLC_STAGES 3   // with 3 B buffers: kernel pair 34.9 -> 34.6 us vs 4 stages / 2 buffers
#endif
constexpr int STAGES = KVLC_STAGES;
constexpr float LAZY = 8.f;
// The lo halves of the PV B operand (p s - hi, ~2^-11 p s) go into their own MMA column
// scaled by PV_LO_SCALE and are unscaled in warp_store: with the fp16-subnormal code
// operands (c 4^j 2^-24) the unscaled lo products sat at the bottom of the tensor core's
// product range and lost low-order bits (KVLC_PV_LO_SCALE A/B, tools/decode_err_diag.py)
#ifndef KVLC_PV_LO_SCALE
#define KVLC_PV_LO_SCALE 1.f
#endif
constexpr float PV_LO_SCALE = KVLC_PV_LO_SCALE;
#ifndef KVLC_BBUF
#define KVLC_BBUF 3
#endif
constexpr int NBUF = KVLC_BBUF;   // B-operand buffers: a warp refills a buffer once every warp is
                                  // done with the chunk NBUF back (static shared memory <= 48 KB)

template <int NG>
struct WarpState {
  static constexpr bool HILO = NG <= 4;
  static constexpr int NH = HILO ? 1 : 2;
  float m[NH];      // reference point of p (log2 units)
  float mt[NH];     // true running max
  float l[NH], z[NH];
  float acc[8][4];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int e = 0; e < NH; ++e) {
      m[e] = -INFINITY;
      mt[e] = -INFINITY;
      l[e] = 0.f;
      z[e] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  }
};

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// Centring of the PV accumulator.  mma.sync accumulates in fp32 rounding toward zero
// (tools/microbench/mma_rounding.cu: +0.6 ulp added 1000 times to 1.0 leaves 1.0), and the
// accumulated sum p s code is all-positive while the output is the small difference
// sum p s code + sum p z (codes 0..3, z the row minimum): at 32k tokens the truncation
// bias, magnified by that cancellation, reached 1.6e-3 of max|out| (T4 is 1e-3).  So
// after each chunk the accumulator drops 3/2 sum p s (the codes become c - 3/2, zero
// mean) and the zero term accumulates the row midpoint z' = z + 3/2 s instead of z:
// both sums stay small and the truncation acts on small values.
// ps: this lane's sum of p s of the chunk per column group e (heads t / 2t + e).
#ifndef KVLC_CENTRE
#define KVLC_CENTRE 1
#endif
constexpr bool CENTRE = KVLC_CENTRE;
template <int NG>
__device__ __forceinline__ void centre_acc(WarpState<NG>& st, float (&ps)[WarpState<NG>::NH]) {
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
#pragma unroll
  for (int e = 0; e < NH; ++e) {
    ps[e] += __shfl_xor_sync(0xffffffffu, ps[e], 4);
    ps[e] += __shfl_xor_sync(0xffffffffu, ps[e], 8);
    ps[e] += __shfl_xor_sync(0xffffffffu, ps[e], 16);
  }
#pragma unroll
  for (int mv = 0; mv < 8; ++mv)
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      // row factor 4^j 2^-24 of the fp16-subnormal codes, j = 2 (mv & 1) + rr
      const float f = -1.5f / code_unscale(2 * (mv & 1) + rr);
      if (HILO) {
        st.acc[mv][2 * rr] = fmaf(f, ps[0], st.acc[mv][2 * rr]);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) st.acc[mv][2 * rr + e] = fmaf(f, ps[e], st.acc[mv][2 * rr + e]);
      }
    }
}

// One chunk of one unit in shared memory: the bytes of the global layouts.
struct ChunkStage {
  uint4 k[WARPS][32][2];   // fragment-native K words of warp slice w, lane l: words 0-3 / 4-7
  uint4 v[WARPS][32][2];   // V words
  uint16_t vs[128], vz[128], ks[128], kz[128];   // fp16 V scale / zero per token, K per channel
};

struct QuantSmem {
  ChunkStage stage[STAGES];
  uint4 bq[NBUF][4][32];   // [buf][k-tile pair][lane]: (b0, b1 of kt = 2p, b0, b1 of kt = 2p+1)
  uint4 bl[NBUF][4][32];   // low parts (groups of > 4 heads)
  float4 zt[NBUF][8];      // [buf][column g] -> partial zero terms of the 4 warps
  uint64_t full[NBUF];     // 4 warp arrivals: every share of the buffer's B is written
  uint64_t empty[NBUF];    // 4 warp arrivals: every warp is done reading the buffer
  uint64_t sfull[STAGES];  // bulk-copy transaction count: the stage's chunk has landed
  uint64_t sempty[STAGES]; // 4 warp arrivals: the stage's chunk is consumed
};

// CTA-scope mbarriers between the 4 warps of a quantized split (one elected lane per
// warp arrives after __syncwarp, so the whole warp's shared-memory writes are released).
__device__ __forceinline__ void qb_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void qb_arrive(uint64_t* bar, int lane) {
  __syncwarp();
  if (lane == 0)
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void qb_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

union SplitSmem {
  QuantSmem quant;
  float rec[WARPS * 8 * REC];
  float corr[8 * D + WARPS * 2 * 8 * HALF + WARPS * 2 * 8 + 2 * 8];  // run_corr_unit, NG <= 8
};

// Thread 0: chunk cb (absolute) into stage `st`, completion on `bar`.
__device__ __forceinline__ void issue_chunk(const kvlc_cache& c, size_t cb, ChunkStage& st, uint64_t* bar) {
  tc::mbar_expect_tx(bar, (uint32_t)sizeof(ChunkStage));
  tc::bulk_g2s(st.k, c.kcodes + cb * 1024, 4096, bar);
  tc::bulk_g2s(st.v, c.vcodes + cb * 1024, 4096, bar);
  tc::bulk_g2s(st.vs, c.vscale + cb * 128, 256, bar);
  tc::bulk_g2s(st.vz, c.vzero + cb * 128, 256, bar);
  tc::bulk_g2s(st.ks, c.kscale + cb * 128, 256, bar);
  tc::bulk_g2s(st.kz, c.kzero + cb * 128, 256, bar);
}

// Builds this warp's share (k-tiles 2w, 2w+1) of a chunk's B operand from its stage.
//  HILO: column n = g holds head g>>1: the hi part for even g, the lo part
//        (exact FMA residual q*s - hi) for odd g.
//  else: column n = g holds head g (hi in bq, lo in bl).
template <int NG>
__device__ __forceinline__ void build_b(QuantSmem& sm, int buf, const ChunkStage& st,
                                        const uint32_t (&qs)[4], int warp, int lane) {
  constexpr bool HILO = NG <= 4;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t* ks = reinterpret_cast<const uint32_t*>(st.ks + 32 * warp);
  const uint32_t* kz = reinterpret_cast<const uint32_t*>(st.kz + 32 * warp);
  uint32_t b[4], bl[4];
  float zp = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // i = 2e + k: channels 32w + 16e + 2t + {0,1} (+8 for k = 1)
    const int pair = 8 * (i >> 1) + t + 4 * (i & 1);
    const __half2 qv = u2h(qs[i]), sv = u2h(ks[pair]);
    const __half2 hi = __hmul2(qv, sv);
    if (HILO) {
      const uint32_t neg = (g & 1) ? (h2u(hi) ^ 0x80008000u) : 0u;
      b[i] = h2u(__hfma2(qv, sv, u2h(neg)));
    } else {
      b[i] = h2u(hi);
      bl[i] = h2u(__hfma2(qv, sv, __hneg2(hi)));
    }
    const float2 qf = __half22float2(qv), zf = __half22float2(u2h(kz[pair]));
    zp = fmaf(qf.x, zf.x, zp);
    zp = fmaf(qf.y, zf.y, zp);
  }
  sm.bq[buf][warp][lane] = make_uint4(b[0], b[1], b[2], b[3]);
  if (!HILO) sm.bl[buf][warp][lane] = make_uint4(bl[0], bl[1], bl[2], bl[3]);
  zp += __shfl_xor_sync(0xffffffffu, zp, 1);
  zp += __shfl_xor_sync(0xffffffffu, zp, 2);
  if (t == 0) reinterpret_cast<float*>(&sm.zt[buf][g])[warp] = zp;
}

// One 128-token chunk, this warp's 32-token slice (tokens 32w .. 32w+31).
// K word kt of lane (g, t) holds channels 16kt+2t+{0,8,1,9} in bytes 0..3 and
// tokens 32w+4g+j at bits 2j; V word 4mt+p holds tokens 32w+8t+2mt+{0,1,4,5}
// in bytes 0..3 and channels 32p+8j+g at bits 2j.
template <int NG, int EXTRA>
__device__ __forceinline__ void quant_chunk(const ChunkStage& stg, const QuantSmem& sm, int buf,
                                            WarpState<NG>& st, int warp, int lane) {
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
  constexpr bool QK_LO = !HILO && (EXTRA & 1);
  constexpr bool PV_LO = !HILO && (EXTRA & 2);
  const int g = lane >> 2, t = lane & 3;

  float zt[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) {
    const float4 zz = sm.zt[buf][HILO ? 2 * t : 2 * t + e];
    zt[e] = ((zz.x + zz.y) + (zz.z + zz.w)) * C0;
  }

  // ---- Q K^T over the slice's 2 token tiles ----
  float cq[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cq[i][j] = 0.f;
  {
    const uint4 k0 = stg.k[warp][lane][0], k1 = stg.k[warp][lane][1];
    const uint32_t kw[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint4 b = sm.bq[buf][p][lane];
      uint4 bl = make_uint4(0u, 0u, 0u, 0u);
      if (QK_LO) bl = sm.bl[buf][p][lane];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t x = kw[2 * p + e], y = code_hi(x);
        const uint32_t b0 = e ? b.z : b.x, b1 = e ? b.w : b.y;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const uint32_t a0 = code_h2(x, 2 * mt), a1 = code_h2(x, 2 * mt + 1);
          const uint32_t a2 = code_h2(y, 2 * mt), a3 = code_h2(y, 2 * mt + 1);
          mma_f16(cq[mt], a0, a1, a2, a3, b0, b1);
          if (QK_LO) mma_f16(cq[mt], a0, a1, a2, a3, e ? bl.z : bl.x, e ? bl.w : bl.y);
        }
      }
    }
  }

  // ---- online softmax: thread holds tokens 32w + 4g + (2mt + r) ----
  float cmax[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) cmax[e] = -INFINITY;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float F = code_unscale(2 * mt + r) * C0;
      if (HILO) {
        const float v = fmaf(cq[mt][2 * r] + cq[mt][2 * r + 1], F, zt[0]);
        cq[mt][2 * r] = v;
        cmax[0] = fmaxf(cmax[0], v);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float v = fmaf(cq[mt][2 * r + e], F, zt[e]);
          cq[mt][2 * r + e] = v;
          cmax[e] = fmaxf(cmax[e], v);
        }
      }
    }
  }
  bool grow = false;
  float mref[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) {
    float m = cmax[e];
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
    st.mt[e] = fmaxf(st.mt[e], m);
    // move the reference point only when p would exceed 2^LAZY
    mref[e] = m > st.m[e] + LAZY ? m : st.m[e];
    grow |= mref[e] != st.m[e];
  }
  if (__any_sync(0xffffffffu, grow)) {
    float sc[NH];
#pragma unroll
    for (int e = 0; e < NH; ++e) {
      sc[e] = fast_exp2(st.m[e] - mref[e]);   // exp2(-inf) = 0 on the first chunk
      st.m[e] = mref[e];
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
  }
  const uint2 vs = reinterpret_cast<const uint2*>(stg.vs + 32 * warp)[g];
  const uint2 vz = reinterpret_cast<const uint2*>(stg.vz + 32 * warp)[g];
  const float2 s01 = __half22float2(u2h(vs.x)), s23 = __half22float2(u2h(vs.y));
  const float2 z01 = __half22float2(u2h(vz.x)), z23 = __half22float2(u2h(vz.y));
  const float svs[4] = {s01.x, s01.y, s23.x, s23.y}, svz[4] = {z01.x, z01.y, z23.x, z23.y};
  uint32_t bp[2][2], bpl[2][2];
  float ps[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) ps[e] = 0.f;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float sv = svs[2 * mt + r], zv = CENTRE ? fmaf(1.5f, svs[2 * mt + r], svz[2 * mt + r]) : svz[2 * mt + r];  // z' (centre_acc)
      if (HILO) {
        const float p = fast_exp2(cq[mt][2 * r] - st.m[0]);
        st.l[0] += p;
        st.z[0] = fmaf(p, zv, st.z[0]);
        const float pv = p * sv;
        ps[0] += pv;
        // hi: pv truncated to 11 significant bits (fp16-exact), lo: the exact remainder
        #ifdef KVLC_HI_RN
        const float hi = __half2float(__float2half_rn(pv));
#else
        const float hi = __uint_as_float(__float_as_uint(pv) & 0xffffe000u);
#endif
        bp[mt][r] = movm_t(h2u(__floats2half2_rn(hi, (pv - hi) * PV_LO_SCALE)));
      } else {
        const float p0 = fast_exp2(cq[mt][2 * r] - st.m[0]);
        const float p1 = fast_exp2(cq[mt][2 * r + 1] - st.m[1]);
        st.l[0] += p0;
        st.l[1] += p1;
        st.z[0] = fmaf(p0, zv, st.z[0]);
        st.z[1] = fmaf(p1, zv, st.z[1]);
        const float a0 = p0 * sv, a1 = p1 * sv;
        const __half2 hh = __floats2half2_rn(a0, a1);
        bp[mt][r] = movm_t(h2u(hh));
        if (PV_LO) {
          const float2 hf = __half22float2(hh);
          bpl[mt][r] = movm_t(h2u(__floats2half2_rn(a0 - hf.x, a1 - hf.y)));
          ps[0] += a0;
          ps[1] += a1;
        } else {  // the MMA sees fp16(p s) only
          const float2 hf = __half22float2(hh);
          ps[0] += hf.x;
          ps[1] += hf.y;
        }
      }
    }
  }

  // ---- P V: 8 channel tiles x the slice's 2 token tiles ----
  const uint4 v0 = stg.v[warp][lane][0], v1 = stg.v[warp][lane][1];
  const uint32_t vw[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint32_t x = vw[4 * mt + p], y = code_hi(x);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int mv = 2 * p + h;
        const uint32_t a0 = code_h2(x, 2 * h), a1 = code_h2(x, 2 * h + 1);
        const uint32_t a2 = code_h2(y, 2 * h), a3 = code_h2(y, 2 * h + 1);
        mma_f16(st.acc[mv], a0, a1, a2, a3, bp[mt][0], bp[mt][1]);
        if (PV_LO) mma_f16(st.acc[mv], a0, a1, a2, a3, bpl[mt][0], bpl[mt][1]);
      }
    }
  }
  if (CENTRE) centre_acc<NG>(st, ps);
}

// Writes this warp's record (m_ref, l, m_true, -, y[c]) per head into shared memory.
// Quantized rows: channel 16mv + g + 8r with factor 2^24 4^-(2(mv&1)+r), plus
// the value zero term; residual rows: channel 16mv + g + 8r, no factor.
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
      r[2] = st.mt[e];
    }
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        float v = HILO ? (QUANT ? fmaf(st.acc[mv][2 * rr + 1], 1.f / PV_LO_SCALE, st.acc[mv][2 * rr])
                                : st.acc[mv][2 * rr] + st.acc[mv][2 * rr + 1])
                       : st.acc[mv][2 * rr + e];
        if (QUANT) v = fmaf(v, code_unscale(2 * (mv & 1) + rr), st.z[e]);
        r[4 + 16 * mv + g + 8 * rr] = v;
      }
    }
  }
}

// Merges the WARPS per-warp records in shared memory into one global record per head.
// (the caller has synchronised after warp_store)
template <int NG>
__device__ __forceinline__ void cta_merge(float* sm, float* out) {
  __shared__ float wts[NG][WARPS];
  __shared__ float hdr[NG][4];
  if (threadIdx.x < NG) {
    const int h = threadIdx.x;
    float M = -INFINITY, Mt = -INFINITY, l = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      M = fmaxf(M, sm[(w * NG + h) * REC]);
      Mt = fmaxf(Mt, sm[(w * NG + h) * REC + 2]);
    }
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const float mw = sm[(w * NG + h) * REC];
      const float wt = mw == -INFINITY ? 0.f : exp2f(mw - M);
      wts[h][w] = wt;
      l = fmaf(wt, sm[(w * NG + h) * REC + 1], l);
    }
    hdr[h][0] = M;
    hdr[h][1] = l;
    hdr[h][2] = Mt;
    hdr[h][3] = 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NG * (D / 4 + 1); i += THREADS) {
    const int h = i / (D / 4 + 1), k4 = i % (D / 4 + 1);
    float4 v;
    if (k4 == 0) {
      v = make_float4(hdr[h][0], hdr[h][1], hdr[h][2], 0.f);
    } else {
      v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const float wt = wts[h][w];
        const float4 y = reinterpret_cast<const float4*>(sm + (w * NG + h) * REC)[k4];
        v.x = fmaf(wt, y.x, v.x);
        v.y = fmaf(wt, y.y, v.y);
        v.z = fmaf(wt, y.z, v.z);
        v.w = fmaf(wt, y.w, v.w);
      }
    }
    reinterpret_cast<float4*>(out + h * REC)[k4] = v;
  }
}

// A quantized split: chunks [lo, hi) of one unit.
template <int NG, int EXTRA>
__device__ __forceinline__ void run_quant(const DecArgs& a, int unit, int split, SplitSmem& sm) {
  const kvlc_cache& c = a.c;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr bool HILO = NG <= 4;
  WarpState<NG> st;
  st.init();
  const int lo = a.chunk_lo + split * a.cpc;
  const int cap_hi = min(min(a.chunk_hi, c.max_chunks), lo + a.cpc);  // no memory read
  const size_t cb0 = (size_t)unit * c.max_chunks;
  QuantSmem& q = sm.quant;
  if (threadIdx.x < 2 * NBUF) qb_init(threadIdx.x < NBUF ? &q.full[threadIdx.x] : &q.empty[threadIdx.x - NBUF], WARPS);
  // prologue: chunks 0 .. STAGES-2 (relative) requested before the sequence length and q
  // arrive, so the round trips overlap; bounded by the cache capacity (always allocated),
  // only chunks below the sequence's count are consumed, the rest drained at the end
  const int n_pro = max(0, min(STAGES - 1, cap_hi - lo));
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&q.sfull[s], 1);
      tc::mbar_init(&q.sempty[s], WARPS);
    }
    tc::mbar_fence_init();
    for (int s = 0; s < n_pro; ++s) issue_chunk(c, cb0 + lo + s, q.stage[s], &q.sfull[s]);
  }
  __syncthreads();  // barriers initialised before any warp waits or arrives
  // the chunk count and q may come from a programmatic-launch predecessor (a flush,
  // kvlc_stage_input): both are read after the wait, their loads issued together
  griddep_wait();
  const int n_ch = min(c.n_chunks[b], a.chunk_hi);
  // q (fp16, exact from bf16) for this warp's B share: column n = g,
  // channels 32w + 16e + 2t + {0,1} (+8)
  uint32_t raw[4];
  {
    const int head = HILO ? (g >> 1) : g;
    const bool valid = head < NG;
    const uint32_t* qp = reinterpret_cast<const uint32_t*>(
        a.q + ((size_t)b * c.Hq + (size_t)kvh * NG + (valid ? head : 0)) * D);
#pragma unroll
    for (int i = 0; i < 4; ++i) raw[i] = valid ? __ldg(qp + 16 * warp + 8 * (i >> 1) + t + 4 * (i & 1)) : 0u;
  }
  const int hi = min(n_ch, lo + a.cpc);
  const int n = max(0, hi - lo);
  if (n > 0) {
    uint32_t qs[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      qs[i] = h2u(__floats2half2_rn(__uint_as_float(raw[i] << 16), __uint_as_float(raw[i] & 0xffff0000u)));
    tc::mbar_wait(&q.sfull[0], 0u);
#ifndef KVLC_PROBE_NOMATH  // probe build: the stream and barriers without the math (timing only)
    build_b<NG>(q, 0, q.stage[0], qs, warp, lane);
#endif
    qb_arrive(&q.full[0], lane);
    for (int k = 0; k < n; ++k) {
      const int buf = k % NBUF, s_cur = k % STAGES;
      qb_wait(&q.full[buf], (uint32_t)(k / NBUF) & 1u);   // every share of chunk k's B
      // every warp has consumed chunk k-1 (its B share of chunk k follows that): refill its stage
      if (threadIdx.x == 0 && k + STAGES - 1 < n) {
        const int j = k + STAGES - 1, s = j % STAGES;
        if (k >= 1) tc::mbar_wait(&q.sempty[s], (uint32_t)((k - 1) / STAGES) & 1u);
        issue_chunk(c, cb0 + lo + j, q.stage[s], &q.sfull[s]);
      }
#ifndef KVLC_PROBE_NOMATH
      quant_chunk<NG, EXTRA>(q.stage[s_cur], q, buf, st, warp, lane);
#endif
      qb_arrive(&q.sempty[s_cur], lane);
      qb_arrive(&q.empty[buf], lane);
      if (k + 1 < n) {
        const int nb = (k + 1) % NBUF, s_next = (k + 1) % STAGES;
        tc::mbar_wait(&q.sfull[s_next], (uint32_t)((k + 1) / STAGES) & 1u);
        if (k + 1 >= NBUF) qb_wait(&q.empty[nb], (uint32_t)((k + 1) / NBUF - 1) & 1u);  // chunk k+1-NBUF done
#ifndef KVLC_PROBE_NOMATH
        build_b<NG>(q, nb, q.stage[s_next], qs, warp, lane);
#endif
        qb_arrive(&q.full[nb], lane);
      }
    }
  }
  // drain speculative prologue chunks that were not consumed (their bytes land in the
  // record area below)
  if (threadIdx.x == 0)
    for (int j = n; j < n_pro; ++j) tc::mbar_wait(&q.sfull[j % STAGES], (uint32_t)(j / STAGES) & 1u);
  __syncthreads();   // the record area aliases the pipeline buffers
  warp_store<NG, true>(st, sm.rec + warp * NG * REC, lane);
  __syncthreads();
  cta_merge<NG>(sm.rec, a.rec + ((size_t)unit * a.nrec + split) * NG * REC);
}
