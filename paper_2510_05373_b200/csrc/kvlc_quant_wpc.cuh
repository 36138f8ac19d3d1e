// Warp-per-chunk quantized split (included by kvlc_decode.cu after kvlc_quant.cuh).
//
// Same arithmetic as kvlc_quant.cuh (decode_step_blocked's per-block scores /
// max / exp / partial numerators, attention.py:238-247), different work split:
// a warp owns WHOLE chunks (warp w of a split takes chunks lo + w, lo + w + 4,
// ...), so
//   * the QK^T B operand of a chunk (q' = q * s_k, fp16 hi/lo) is built by the
//     warp that uses it, in registers: no shared-memory exchange and no
//     full / empty barriers between the warps (the slice layout waited on its
//     peers' B shares every chunk: 10.6 % of the stall samples, r01j);
//   * the zero term zt = q . z_k is one m16n8k16 MMA per k-tile with A = the
//     chunk's z_k in every row and B = q: no per-lane fp32 loop, no shuffles;
//   * the softmax bookkeeping (row max across lanes, the lazy-rescale vote) runs
//     once per 128 tokens instead of once per 32;
//   * each warp streams its own chunks as half-chunks (K codes + K scale / zero,
//     then V codes + V scale / zero, 4.5 KB each) through a private ring of 3
//     half-stages (TMA bulk copies, one transaction-count mbarrier per stage),
//     refilled by its lane 0 as soon as the warp has read a half: one chunk in
//     flight per warp, 54 KB of ring per CTA, 4 CTAs (16 warps) per SM for groups
//     of <= 4 heads (q then lives in shared memory, 128 registers per thread).
// Measured against the one-slice-per-warp split (r02 traces, config 2): 30 % fewer
// instructions per chunk (1265 vs ~1800).
#pragma once

constexpr int WPC_RING = 3;  // half-stages per warp: K_i, V_i, K_{i+1} resident / in flight

struct HalfStage {
  uint4 w[WARPS][32][2];   // code words of the 4 32-token slices (fragment-native layouts)
  uint16_t s[128], z[128]; // fp16 scale / zero: per channel (K half) or per token (V half)
};
static_assert(sizeof(HalfStage) == 4608, "half-stage = 4 KB codes + 512 B metadata");

constexpr int QSM_STRIDE = 68;  // words per head of the shared q copy (64 + 4: conflict-free)

struct WpcSmem {
  HalfStage ring[WARPS][WPC_RING];
  uint64_t full[WARPS][WPC_RING];
  uint32_t qsm[4 * QSM_STRIDE];   // q as fp16 pairs, [head][pair] (groups of <= 4 heads)
};
constexpr size_t WPC_SMEM = sizeof(WpcSmem) > sizeof(float) * WARPS * 8 * REC ? sizeof(WpcSmem)
                                                                                 : sizeof(float) * WARPS * 8 * REC;

// Half j of this warp's chunk sequence: chunk j >> 1, K codes (even j) or V codes (odd j).
// Called by the whole warp: one lane, picked by elect.sync inside the asm, arms the barrier
// and issues the three bulk copies (a divergent `if (lane == 0)` around uniform-datapath
// instructions compiles to a per-instruction ELECT loop).
__device__ __forceinline__ void issue_half(const kvlc_cache& c, size_t cb, int kind, HalfStage& st,
                                           uint64_t* bar) {
  const uint32_t* wsrc = (kind ? c.vcodes : c.kcodes) + cb * 1024;
  const uint16_t* ssrc = (kind ? c.vscale : c.kscale) + cb * 128;
  const uint16_t* zsrc = (kind ? c.vzero : c.kzero) + cb * 128;
  asm volatile(
      "{\n.reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "@p fence.proxy.async.shared::cta;\n"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], 4096, [%0];\n"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5], 256, [%0];\n"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%6], [%7], 256, [%0];\n"
      "}\n" ::"r"(tc::smem_u32(bar)),
      "r"((uint32_t)sizeof(HalfStage)), "r"(tc::smem_u32(st.w)), "l"(wsrc), "r"(tc::smem_u32(st.s)), "l"(ssrc),
      "r"(tc::smem_u32(st.z)), "l"(zsrc)
      : "memory");
}

// q pair i (i = 2 kt + k: channels 16 kt + 2 t + {0,1}, +8 for k = 1) of this lane's head.
template <bool QSM>
__device__ __forceinline__ uint32_t q_pair(const uint32_t (&qs)[16], const uint32_t* qrow, int i, int t) {
  if (QSM) return qrow[8 * (i >> 1) + t + 4 * (i & 1)];
  return qs[i];
}

// QK^T, softmax and PV of one whole chunk (128 tokens = the 4 32-token slices) by one warp.
// kst / vst: the chunk's K and V half-stages; vst is waited for (vbar, vpar) only after the
// scores, so the V half may still be in flight during QK^T.  k_done() runs once every lane
// has read the K half (its slot is refilled while the softmax and PV run).
template <int NG, int EXTRA, bool QSM, class KDone>
__device__ __forceinline__ void wpc_chunk(const HalfStage& kst, const HalfStage& vst, uint64_t* vbar,
                                          uint32_t vpar, const uint32_t (&qs)[16], const uint32_t* qrow,
                                          WarpState<NG>& st, int lane, KDone k_done) {
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
  constexpr bool QK_LO = !HILO && (EXTRA & 1);
  constexpr bool PV_LO = !HILO && (EXTRA & 2);
  const int g = lane >> 2, t = lane & 3;

  // ---- B operand q' = q * s_k (hi / lo) and the zero term q . z_k ----
  const uint32_t* ks = reinterpret_cast<const uint32_t*>(kst.s);
  const uint32_t* kz = reinterpret_cast<const uint32_t*>(kst.z);
  uint32_t bq[8][2], bl[8][2];
  float zc[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t odd = (g & 1) ? 0xffffffffu : 0u;
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) {
    uint32_t zz[2], qq[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int pair = 8 * kt + t + 4 * k;
      qq[k] = q_pair<QSM>(qs, qrow, 2 * kt + k, t);
      const __half2 qv = u2h(qq[k]), sv = u2h(ks[pair]);
      const __half2 hi = __hmul2(qv, sv);
      if (HILO) {
        // even columns: the hi part; odd columns: the exact FMA residual q*s - hi
        bq[kt][k] = h2u(__hfma2(qv, sv, u2h((h2u(hi) ^ 0x80008000u) & odd)));
      } else {
        bq[kt][k] = h2u(hi);
        bl[kt][k] = h2u(__hfma2(qv, sv, __hneg2(hi)));
      }
      zz[k] = kz[pair];
    }
    // every row of A = z_k of the k-tile: C[row][n] = sum_c z_k[c] q[head(n)][c] (exact products)
    mma_f16(zc, zz[0], zz[0], zz[1], zz[1], qq[0], qq[1]);
  }
  // column 2t (+1): head t (HILO, both columns) or heads 2t, 2t+1
  float zt[NH];
  zt[0] = zc[0] * C0;
  if (!HILO) zt[NH - 1] = zc[1] * C0;

  // ---- Q K^T over the 4 slices x 2 token tiles ----
  float cq[4][2][4];
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) cq[s][i][j] = 0.f;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint4 k0 = kst.w[s][lane][0], k1 = kst.w[s][lane][1];
    const uint32_t kw[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      const uint32_t x = kw[kt], y = code_hi(x);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const uint32_t a0 = code_h2(x, 2 * mt), a1 = code_h2(x, 2 * mt + 1);
        const uint32_t a2 = code_h2(y, 2 * mt), a3 = code_h2(y, 2 * mt + 1);
        mma_f16(cq[s][mt], a0, a1, a2, a3, bq[kt][0], bq[kt][1]);
        if (QK_LO) mma_f16(cq[s][mt], a0, a1, a2, a3, bl[kt][0], bl[kt][1]);
      }
    }
  }

  k_done();

  // ---- online softmax over the chunk: thread holds tokens 32s + 4g + (2mt + r) ----
  float cmax[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) cmax[e] = -INFINITY;
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float F = code_unscale(2 * mt + r) * C0;
        if (HILO) {
          const float v = fmaf(cq[s][mt][2 * r] + cq[s][mt][2 * r + 1], F, zt[0]);
          cq[s][mt][2 * r] = v;
          cmax[0] = fmaxf(cmax[0], v);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float v = fmaf(cq[s][mt][2 * r + e], F, zt[e]);
            cq[s][mt][2 * r + e] = v;
            cmax[e] = fmaxf(cmax[e], v);
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
      sc[e] = fast_exp2(st.m[e] - mref[e]);  // exp2(-inf) = 0 on the first chunk
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

  // ---- p (value scale folded in) as PV B fragments, then P V per slice ----
  tc::mbar_wait(vbar, vpar);
  float ps[NH];
#pragma unroll
  for (int e = 0; e < NH; ++e) ps[e] = 0.f;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint2 vs = reinterpret_cast<const uint2*>(vst.s + 32 * s)[g];
    const uint2 vz = reinterpret_cast<const uint2*>(vst.z + 32 * s)[g];
    const float2 s01 = __half22float2(u2h(vs.x)), s23 = __half22float2(u2h(vs.y));
    const float2 z01 = __half22float2(u2h(vz.x)), z23 = __half22float2(u2h(vz.y));
    const float svs[4] = {s01.x, s01.y, s23.x, s23.y}, svz[4] = {z01.x, z01.y, z23.x, z23.y};
    uint32_t bp[2][2], bpl[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float sv = svs[2 * mt + r], zv = CENTRE ? fmaf(1.5f, svs[2 * mt + r], svz[2 * mt + r]) : svz[2 * mt + r];  // z' (centre_acc)
        if (HILO) {
          const float p = fast_exp2(cq[s][mt][2 * r] - st.m[0]);
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
          const float p0 = fast_exp2(cq[s][mt][2 * r] - st.m[0]);
          const float p1 = fast_exp2(cq[s][mt][2 * r + 1] - st.m[1]);
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
    const uint4 v0 = vst.w[s][lane][0], v1 = vst.w[s][lane][1];
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
  }
  if (CENTRE) centre_acc<NG>(st, ps);
}

// A quantized split, warp per chunk: chunks [lo, hi) of one unit, warp w takes lo + w + 4i.
// Half j of the warp's sequence (chunk j >> 1, K / V by j & 1) lives in ring slot j % 3.
template <int NG, int EXTRA>
__device__ __forceinline__ void run_quant_wpc(const DecArgs& a, int unit, int split, WpcSmem& q, float* rec_sm) {
  const kvlc_cache& c = a.c;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr bool HILO = NG <= 4;
#ifndef KVLC_WPC_QSM
#define KVLC_WPC_QSM 1
#endif
  // q from shared memory: frees registers for the pipeline (also at 3 CTAs per SM: 34.7 vs 35.0 us
  // with q in registers, config 2)
  constexpr bool QSM = HILO && KVLC_WPC_QSM;
  WarpState<NG> st;
  st.init();
  const int lo = a.chunk_lo + split * a.cpc;
  const int cap_hi = min(min(a.chunk_hi, c.max_chunks), lo + a.cpc);  // no memory read
  const size_t cb0 = (size_t)unit * c.max_chunks + lo + warp;         // this warp's first chunk
  const int cap_n = cap_hi - lo > warp ? (cap_hi - lo - warp + 3) / 4 : 0;
  // prologue: the warp's first 3 halves requested before the sequence length and q arrive
  // (bounded by the cache capacity, always allocated; unconsumed ones drained below)
  const int n_pro = min(WPC_RING, 2 * cap_n);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < WPC_RING; ++s) tc::mbar_init(&q.full[warp][s], 1);
    tc::mbar_fence_init();
  }
  __syncwarp();
  for (int j = 0; j < n_pro; ++j) issue_half(c, cb0 + 4 * (j >> 1), j & 1, q.ring[warp][j], &q.full[warp][j]);
  // the chunk count and q may come from a programmatic-launch predecessor (a flush,
  // kvlc_stage_input): both are read after the wait, their loads issued together
  griddep_wait();
  PH_STAMP(0);
  const int n_ch = min(c.n_chunks[b], a.chunk_hi);
  const uint32_t* qrow = q.qsm + (g >> 1) * QSM_STRIDE;
  uint32_t qs[16];
  {
    const uint32_t* qp = reinterpret_cast<const uint32_t*>(a.q + ((size_t)b * c.Hq + (size_t)kvh * NG) * D);
    if (QSM) {
      // the unit's NG heads as fp16 pairs (exact from bf16), [head][pair]
      for (int i = threadIdx.x; i < 4 * 64; i += THREADS) {
        const int h = i >> 6, pr = i & 63;
        const uint32_t r = h < NG ? __ldg(qp + h * (D / 2) + pr) : 0u;
        q.qsm[h * QSM_STRIDE + pr] =
            h2u(__floats2half2_rn(__uint_as_float(r << 16), __uint_as_float(r & 0xffff0000u)));
      }
    } else {
      const int head = HILO ? (g >> 1) : g;
      const bool valid = head < NG;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t r = valid ? __ldg(qp + head * (D / 2) + 8 * (i >> 1) + t + 4 * (i & 1)) : 0u;
        qs[i] = h2u(__floats2half2_rn(__uint_as_float(r << 16), __uint_as_float(r & 0xffff0000u)));
      }
    }
  }
  __syncthreads();  // barriers initialised, shared q written
  PH_STAMP(1);
  const int hi = min(n_ch, lo + a.cpc);
  const int n = max(0, hi - lo);
  const int my_n = n > warp ? (n - warp + 3) / 4 : 0;
  // refill of a consumed slot with half j (if the warp has it)
  auto refill = [&](int j) {
    __syncwarp();  // every lane has read the slot (issue_half fences it for the async proxy)
    if (j < 2 * my_n) issue_half(c, cb0 + 4 * (j >> 1), j & 1, q.ring[warp][j % WPC_RING], &q.full[warp][j % WPC_RING]);
  };
  for (int i = 0; i < my_n; ++i) {
    const int jk = 2 * i, jv = 2 * i + 1;
    const int sk = jk % WPC_RING, sv = jv % WPC_RING;
    tc::mbar_wait(&q.full[warp][sk], (uint32_t)(jk / WPC_RING) & 1u);
#ifndef KVLC_PROBE_NOMATH  // probe build: the stream without the math (timing only)
    // K_i's slot takes V_{i+1} after QK^T, V_i's slot takes K_{i+2} after PV: one chunk of
    // lead for both halves
    wpc_chunk<NG, EXTRA, QSM>(q.ring[warp][sk], q.ring[warp][sv], &q.full[warp][sv],
                              (uint32_t)(jv / WPC_RING) & 1u, qs, qrow, st, lane,
                              [&] { refill(jk + WPC_RING); });
#else
    refill(jk + WPC_RING);
    tc::mbar_wait(&q.full[warp][sv], (uint32_t)(jv / WPC_RING) & 1u);
#endif
    refill(jv + WPC_RING);
  }
  // drain speculative prologue halves that were not consumed (the record area aliases the ring)
  if (lane == 0) {
    for (int j = 2 * my_n; j < n_pro; ++j) tc::mbar_wait(&q.full[warp][j], 0u);
#pragma unroll
    for (int s = 0; s < WPC_RING; ++s)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(tc::smem_u32(&q.full[warp][s])) : "memory");
  }
  if (a.rps == 4) {  // one record per warp, straight to global memory: no CTA barrier or merge
    __syncwarp();
    warp_store<NG, true>(st, a.rec + ((size_t)unit * a.nrec + 4 * split + warp) * NG * REC, lane);
    return;
  }
  __syncthreads();
  PH_STAMP(2);
  warp_store<NG, true>(st, rec_sm + warp * NG * REC, lane);
  __syncthreads();
  cta_merge<NG>(rec_sm, a.rec + ((size_t)unit * a.nrec + split) * NG * REC);
}
