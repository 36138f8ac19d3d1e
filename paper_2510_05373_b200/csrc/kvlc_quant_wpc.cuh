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
//   * each warp streams its own chunks through a private 2-stage ring (TMA bulk
//     copies, one transaction-count mbarrier per stage), refilled by its lane 0
//     as soon as the warp has read a stage: no cross-warp stage release.
// Shared memory is 72 KB per CTA (dynamic), 3 CTAs per SM.
#pragma once

constexpr int WPC_STAGES = 2;

struct WpcSmem {
  ChunkStage stage[WARPS][WPC_STAGES];
  uint64_t full[WARPS][WPC_STAGES];
};
constexpr size_t WPC_SMEM = sizeof(WpcSmem) > sizeof(float) * WARPS * 8 * REC ? sizeof(WpcSmem)
                                                                                 : sizeof(float) * WARPS * 8 * REC;

// One whole chunk (128 tokens = the 4 32-token slices of the layout) by one warp.
// qs: q as fp16 pairs, B-fragment order: qs[2 kt + k] = channels 16 kt + 2 t + {0,1} (+8 for k = 1)
// of head g >> 1 (HILO) or g.
template <int NG, int EXTRA>
__device__ __forceinline__ void wpc_chunk(const ChunkStage& stg, const uint32_t (&qs)[16], WarpState<NG>& st,
                                          int lane) {
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
  constexpr bool QK_LO = !HILO && (EXTRA & 1);
  constexpr bool PV_LO = !HILO && (EXTRA & 2);
  const int g = lane >> 2, t = lane & 3;

  // ---- B operand q' = q * s_k (hi / lo) and the zero term q . z_k ----
  const uint32_t* ks = reinterpret_cast<const uint32_t*>(stg.ks);
  const uint32_t* kz = reinterpret_cast<const uint32_t*>(stg.kz);
  uint32_t bq[8][2], bl[8][2];
  float zc[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t odd = (g & 1) ? 0xffffffffu : 0u;
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) {
    uint32_t zz[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int pair = 8 * kt + t + 4 * k;
      const __half2 qv = u2h(qs[2 * kt + k]), sv = u2h(ks[pair]);
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
    mma_f16(zc, zz[0], zz[0], zz[1], zz[1], qs[2 * kt], qs[2 * kt + 1]);
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
    const uint4 k0 = stg.k[s][lane][0], k1 = stg.k[s][lane][1];
    const uint32_t kw[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      const uint32_t x = kw[kt], y = x >> 8;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const uint32_t a0 = code_h2(x, 2 * mt), a1 = code_h2(x, 2 * mt + 1);
        const uint32_t a2 = code_h2(y, 2 * mt), a3 = code_h2(y, 2 * mt + 1);
        mma_f16(cq[s][mt], a0, a1, a2, a3, bq[kt][0], bq[kt][1]);
        if (QK_LO) mma_f16(cq[s][mt], a0, a1, a2, a3, bl[kt][0], bl[kt][1]);
      }
    }
  }

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
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const uint2 vs = reinterpret_cast<const uint2*>(stg.vs + 32 * s)[g];
    const uint2 vz = reinterpret_cast<const uint2*>(stg.vz + 32 * s)[g];
    const float2 s01 = __half22float2(u2h(vs.x)), s23 = __half22float2(u2h(vs.y));
    const float2 z01 = __half22float2(u2h(vz.x)), z23 = __half22float2(u2h(vz.y));
    const float svs[4] = {s01.x, s01.y, s23.x, s23.y}, svz[4] = {z01.x, z01.y, z23.x, z23.y};
    uint32_t bp[2][2], bpl[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float sv = svs[2 * mt + r], zv = svz[2 * mt + r];
        if (HILO) {
          const float p = fast_exp2(cq[s][mt][2 * r] - st.m[0]);
          st.l[0] += p;
          st.z[0] = fmaf(p, zv, st.z[0]);
          const float pv = p * sv;
          // hi: pv truncated to 11 significant bits (fp16-exact), lo: the exact remainder
          const float hi = __uint_as_float(__float_as_uint(pv) & 0xffffe000u);
          bp[mt][r] = movm_t(h2u(__floats2half2_rn(hi, pv - hi)));
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
          }
        }
      }
    }
    const uint4 v0 = stg.v[s][lane][0], v1 = stg.v[s][lane][1];
    const uint32_t vw[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const uint32_t x = vw[4 * mt + p], y = x >> 8;
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
}

// A quantized split, warp per chunk: chunks [lo, hi) of one unit, warp w takes lo + w + 4i.
template <int NG, int EXTRA>
__device__ void run_quant_wpc(const DecArgs& a, int unit, int split, WpcSmem& q, float* rec_sm) {
  const kvlc_cache& c = a.c;
  const int b = unit / c.Hkv, kvh = unit % c.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr bool HILO = NG <= 4;
  WarpState<NG> st;
  st.init();
  const int lo = a.chunk_lo + split * a.cpc;
  const int cap_hi = min(min(a.chunk_hi, c.max_chunks), lo + a.cpc);  // no memory read
  const size_t cb0 = (size_t)unit * c.max_chunks + lo + warp;         // this warp's first chunk
  const int cap_n = cap_hi - lo > warp ? (cap_hi - lo - warp + 3) / 4 : 0;
  // prologue: the warp's first WPC_STAGES chunks requested before the sequence length and q
  // arrive (bounded by the cache capacity, always allocated; unconsumed ones drained below)
  const int n_pro = min(WPC_STAGES, cap_n);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < WPC_STAGES; ++s) tc::mbar_init(&q.full[warp][s], 1);
    tc::mbar_fence_init();
    for (int s = 0; s < n_pro; ++s) issue_chunk(c, cb0 + 4 * s, q.stage[warp][s], &q.full[warp][s]);
  }
  __syncwarp();
  // the chunk count and q may come from a programmatic-launch predecessor (a flush,
  // kvlc_stage_input): both are read after the wait, their loads issued together
  griddep_wait();
  const int n_ch = min(c.n_chunks[b], a.chunk_hi);
  uint32_t raw[16];
  {
    const int head = HILO ? (g >> 1) : g;
    const bool valid = head < NG;
    const uint32_t* qp = reinterpret_cast<const uint32_t*>(
        a.q + ((size_t)b * c.Hq + (size_t)kvh * NG + (valid ? head : 0)) * D);
#pragma unroll
    for (int i = 0; i < 16; ++i) raw[i] = valid ? __ldg(qp + 8 * (i >> 1) + t + 4 * (i & 1)) : 0u;
  }
  const int hi = min(n_ch, lo + a.cpc);
  const int n = max(0, hi - lo);
  const int my_n = n > warp ? (n - warp + 3) / 4 : 0;
  if (my_n > 0) {
    // q as fp16 (exact from bf16), B-fragment order
    uint32_t qs[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      qs[i] = h2u(__floats2half2_rn(__uint_as_float(raw[i] << 16), __uint_as_float(raw[i] & 0xffff0000u)));
    for (int i = 0; i < my_n; ++i) {
      const int s = i % WPC_STAGES;
      tc::mbar_wait(&q.full[warp][s], (uint32_t)(i / WPC_STAGES) & 1u);
#ifndef KVLC_PROBE_NOMATH  // probe build: the stream without the math (timing only)
      wpc_chunk<NG, EXTRA>(q.stage[warp][s], qs, st, lane);
#endif
      if (i + WPC_STAGES < my_n) {
        __syncwarp();  // every lane has read the stage
        if (lane == 0) {
          tc::fence_proxy_async();
          issue_chunk(c, cb0 + 4 * (i + WPC_STAGES), q.stage[warp][s], &q.full[warp][s]);
        }
      }
    }
  }
  // drain speculative prologue chunks that were not consumed (the record area aliases the ring)
  if (lane == 0)
    for (int j = my_n; j < n_pro; ++j) tc::mbar_wait(&q.full[warp][j], 0u);
  __syncthreads();
  warp_store<NG, true>(st, rec_sm + warp * NG * REC, lane);
  __syncthreads();
  cta_merge<NG>(rec_sm, a.rec + ((size_t)unit * a.nrec + split) * NG * REC);
}
