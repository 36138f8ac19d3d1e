// Quantized-split path of the fused decode (included by kvlc_decode.cu), on
// the 5th-generation tensor cores (tcgen05, TMEM accumulators, bulk TMA).
//
// A quantized-split CTA (4 warps, thread i) owns chunks [lo, hi) of one
// (b, kv-head) unit.  Per 128-token chunk:
//   * one elected thread streams the chunk (K codes 4 KB, V codes 4 KB, the
//     four 256-B fp16 scale / zero vectors) into an NSTAGE-deep shared-memory
//     ring with cp.async.bulk (TMA), completion on an mbarrier;
//   * thread i expands token i's K row and channel i's V row (2-bit codes ->
//     fp16 pairs, one LOP3 per two codes: the exact subnormals c*4^p*2^-24 of
//     the row-native layout written by kvlc_flush.cu) and stores them into
//     TMEM with tcgen05.st — TMEM lane i is row i of the MMA A operand;
//   * the small B operands live in shared memory: B_QK[c] = q*s_k[c]*4^-p(c)
//     (fp16 hi + lo columns per GQA head; the 4^-p undoes the code's bit-pair
//     weight) and, after the softmax, B_PV[t] = p_t*s_v[t]*4^-p(t); the zero
//     terms q . z_k (keys) and sum_t p_t z_v[t] (values) are per-head scalars
//     computed in fp32;
//   * MMAs are kind::f16, M = 128, N = 16, K = 16 with f32 accumulators in
//     TMEM: D_QK = A_K B_QK (logits), D_PV = A_V B_PV (numerator);
//   * the online softmax keeps one CTA-wide reference point per head (log2
//     units) that moves only when a logit exceeds it by LAZY (rare); each
//     chunk's PV result is drained from TMEM into fp32 registers (the tensor
//     core's f32 accumulation is not carried across chunks).
// Roles and pipeline: see run_quant below.
// Reference: the per-block loop of decode_step_blocked (attention.py:238-247)
// with the block partial (m, l, y) of DecodePartial (attention.py:41-47).
#pragma once



constexpr float LAZY = 6.f;          // reference point moves when p would exceed 2^LAZY
constexpr int NSTAGE = 5;            // chunk ring depth (cp.async lookahead NSTAGE - 2 chunks)
constexpr int MAX_CPC = 64;          // chunks per quantized split (plan_for caps cpc)
constexpr int IFIFO = 8;             // quantized items in flight per CTA (> NSTAGE + 1)
constexpr float QK_SCALE = 256.f;    // B_QK / B_Z prescale (fp16 range use), undone on readback

// TMEM columns (256 allocated per CTA; 2 quantized CTAs per SM)
constexpr uint32_t COL_AK = 0;      // A_K x2 [128 tokens][128 channels] fp16 pairs: 2 x 64 columns
constexpr uint32_t COL_AV = 128;    // A_V    [128 channels][128 tokens]: 64 columns
constexpr uint32_t COL_DQK = 192;   // D_QK   [128 tokens][16] f32
constexpr uint32_t COL_DPV = 208;   // D_PV   [128 channels][16] f32
constexpr uint32_t COL_ONES = 224;  // A_ones [128][16] fp16 2^-24 (key zero term): 8 columns
constexpr uint32_t TMEM_COLS = 256;

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

struct ChunkStage {
  uint4 kc[256];    // K codes: token row r = words 0-3 at uint4 2r + sw(r), words 4-7 at 2r + 1 - sw(r)
  uint4 vc[256];    // V codes: channel row, same swizzle
  uint16_t ks[128], kz[128];  // per channel
  uint16_t vs[128], vz[128];  // per token
};

struct QItem {
  int unit, split, n;  // chunks [chunk_lo + split * cpc, + n) of unit
};

struct TcSmem {
  ChunkStage stage[NSTAGE];
  uint4 bqk[2][256];  // [128 rows][16 cols] fp16 MN-major: cols 0-7 at uint4 r, cols 8-15 at 128 + r
  uint4 bz[2][256];   // key zero-term rows (q z_k), same layout
  uint4 bpv[2][256];  // double-buffered: the MMA of chunk k-1 may still read the other one
  float ob[2][8];     // reference point of chunk k's B_PV [k & 1][head]
  float red[4][8][4];
  float itred[2][4][8][4];  // per-item token-warp totals (l, sum p z_v, true max) [item & 1][warp][head]
  QItem items[IFIFO];       // quantized items of this CTA's chunk stream (FIFO, index & (IFIFO - 1))
  uint16_t qv[IFIFO][8][128];  // their query vectors (bf16, staged by the loaders with cp.async)
  int n_items;              // items popped into the FIFO
  int empty_unit, empty_split;  // loader scratch: a popped item without chunks
  int loaded;               // stream chunks issued into the ring
  int end;                  // stream length once the loaders reached the end of the quantized items
  int next;                 // first non-quantized work item popped by the loaders
  uint64_t mqk, mpv;
  uint32_t tbase;
};

// Residual-window warp state (kvlc_decode.cu run_resid): mma.sync bf16 path.
template <int NG>
struct WarpState {
  static constexpr bool HILO = NG <= 4;
  static constexpr int NH = HILO ? 1 : 2;
  float m[NH];   // reference point of p (log2 units)
  float mt[NH];  // true running max
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

// Writes a residual warp's record (m_ref, l, m_true, -, y[c]) per head into shared memory.
template <int NG>
__device__ __forceinline__ void warp_store(WarpState<NG>& st, float* smrec, int lane) {
  constexpr bool HILO = NG <= 4;
  constexpr int NH = WarpState<NG>::NH;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int e = 0; e < NH; ++e) {
    float l = st.l[e];
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    st.l[e] = l;
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
    for (int mv = 0; mv < 8; ++mv)
#pragma unroll
      for (int rr = 0; rr < 2; ++rr)
        r[4 + 16 * mv + g + 8 * rr] = HILO ? st.acc[mv][2 * rr] + st.acc[mv][2 * rr + 1] : st.acc[mv][2 * rr + e];
  }
}

// Merges the WARPS per-warp records in shared memory into one global record per head.
// (the caller has synchronised after warp_store)
template <int NG, int NW>
__device__ __forceinline__ void cta_merge(float* sm, float* out) {
  __shared__ float wts[NG][NW];
  __shared__ float hdr[NG][4];
  if (threadIdx.x < NG) {
    const int h = threadIdx.x;
    float M = -INFINITY, Mt = -INFINITY, l = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      M = fmaxf(M, sm[(w * NG + h) * REC]);
      Mt = fmaxf(Mt, sm[(w * NG + h) * REC + 2]);
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
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
  for (int i = threadIdx.x; i < NG * (D / 4 + 1); i += blockDim.x) {
    const int h = i / (D / 4 + 1), k4 = i % (D / 4 + 1);
    float4 v;
    if (k4 == 0) {
      v = make_float4(hdr[h][0], hdr[h][1], hdr[h][2], 0.f);
    } else {
      v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < NW; ++w) {
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

// ------------------------------------------------------------ tcgen05 path --

// 2-bit row (8 packed words) -> 64 fp16-pair registers -> TMEM columns [col, col+64)
// of this thread's lane.  Column j = 8w + 4r + p holds the bit pair p of bytes
// r (low half) and r + 2 (high half) of word w.
__device__ __forceinline__ void expand4(const uint4& w, uint32_t* r) {
  const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t y = x[i] >> 8;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      r[8 * i + p] = x[i] & (0x00030003u << (2 * p));
      r[8 * i + 4 + p] = y & (0x00030003u << (2 * p));
    }
  }
}
__device__ __forceinline__ void expand_row(const uint4* rows, int row, uint32_t taddr) {
  const int sw = (row >> 2) & 1;  // 16-B halves swapped on alternate 4-row groups: conflict-free LDS.128
  const uint4 w0 = rows[2 * row + sw], w1 = rows[2 * row + (sw ^ 1)];
  uint32_t r[32];
  expand4(w0, r);
  kvlc::tc::tmem_st32(taddr, r);
  expand4(w1, r);
  kvlc::tc::tmem_st32(taddr + 32, r);
}

__device__ __forceinline__ uint32_t f2h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Row r of an N = 16 B tile: head h's fp16 hi part at column h, lo part
// (exact remainder, rounded) at column LO + h (LO = 4 for <= 4 heads, else 8).
template <int NG>
__device__ __forceinline__ void write_brow(uint4* tile, int r, const float* x) {
  constexpr int NP = NG <= 4 ? 4 : 8;
  float v[NP], lo[NP];
#pragma unroll
  for (int h = 0; h < NP; ++h) v[h] = h < NG ? x[h] : 0.f;
  uint32_t hi2[NP / 2], lo2[NP / 2];
#pragma unroll
  for (int i = 0; i < NP / 2; ++i) {
    hi2[i] = f2h2(v[2 * i], v[2 * i + 1]);
    const float2 hf = __half22float2(*reinterpret_cast<__half2*>(&hi2[i]));
    lo[2 * i] = v[2 * i] - hf.x;
    lo[2 * i + 1] = v[2 * i + 1] - hf.y;
    lo2[i] = f2h2(lo[2 * i], lo[2 * i + 1]);
  }
  if constexpr (NG <= 4) {
    tile[r] = make_uint4(hi2[0], hi2[1], lo2[0], lo2[1]);
  } else {
    tile[r] = make_uint4(hi2[0], hi2[1], hi2[2], hi2[3]);
    tile[128 + r] = make_uint4(lo2[0], lo2[1], lo2[2], lo2[3]);
  }
}

template <int NG>
__device__ __forceinline__ void ld_d(uint32_t taddr, uint32_t* d) {
  if constexpr (NG <= 4) kvlc::tc::tmem_ld8(taddr, d);
  else kvlc::tc::tmem_ld16(taddr, d);
}
template <int NG>
__device__ __forceinline__ void sum_d(const uint32_t* d, float* out) {  // out[h] = hi + lo columns
  constexpr int LO = NG <= 4 ? 4 : 8;
#pragma unroll
  for (int h = 0; h < NG; ++h) out[h] = __uint_as_float(d[h]) + __uint_as_float(d[LO + h]);
}

__device__ __forceinline__ float h2f(uint16_t x) { return __half2float(__ushort_as_half(x)); }

// Optional phase tracing (tools/trace_probe.py; build with -DKVLC_TRACE): clock64
// stamps of token warp 0 / channel warp 4 lane 0 for the first TRACE_CTAS CTAs.
#ifdef KVLC_TRACE
constexpr int TRACE_CTAS = 4, TRACE_K = 32, TRACE_PTS = 28;
__device__ long long g_trace[TRACE_CTAS][TRACE_K + 1][TRACE_PTS];
#define KVLC_STAMP(k, i)                                                                        \
  do {                                                                                          \
    if (blockIdx.x < TRACE_CTAS && (k) < TRACE_K && (threadIdx.x & 127) == 0)                  \
      g_trace[blockIdx.x][(k) < 0 ? TRACE_K : (k)][i] = clock64();                              \
  } while (0)
#define KVLC_STAMP_WARP(k)                                                                      \
  do {                                                                                          \
    if (blockIdx.x < TRACE_CTAS && (k) < TRACE_K && (threadIdx.x & 31) == 0)                   \
      g_trace[blockIdx.x][k][16 + (threadIdx.x >> 5)] = clock64();                              \
  } while (0)
#else
#define KVLC_STAMP_WARP(k) \
  do {                     \
  } while (0)
#define KVLC_STAMP(k, i) \
  do {                   \
  } while (0)
#endif

// Named barriers among the 4 token warps (id 1); id 0 is __syncthreads.
__device__ __forceinline__ void tbar_sync() { asm volatile("barrier.cta.sync 1, 128;\n" ::: "memory"); }
__device__ __forceinline__ bool tbar_or(bool pred) {
  uint32_t r;
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.u32 p, %1, 0;\nbarrier.cta.red.or.pred q, 1, 128, p;\nselp.u32 %0, 1, 0, q;\n}\n"
      : "=r"(r)
      : "r"((uint32_t)pred)
      : "memory");
  return r != 0;
}

__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Named barriers: 1 = token warps (128), 2 = loader warps 6-7 (64), 3 = channel warps (128).
__device__ __forceinline__ void lbar_sync() { asm volatile("barrier.cta.sync 2, 64;\n" ::: "memory"); }
__device__ __forceinline__ void cbar_sync() { asm volatile("barrier.cta.sync 3, 128;\n" ::: "memory"); }

// The quantized work of a persistent split CTA: one continuous chunk stream
// over the quantized items it pops from the global queue.  256 threads:
//   token warps 0-3   (thread = token t of a chunk, TMEM lane t): K-row
//                     expansion into A_K (double-buffered, so chunk k+1's
//                     expansion overlaps the QK MMAs of chunk k), the B_QK /
//                     B_Z rows of chunk k+1 (row = thread index), QK readback,
//                     online softmax, B_PV row t, per-item totals.
//   channel warps 4-7 (thread = channel c, TMEM lane c): PV readback into the
//                     fp32 numerator, V-row expansion into A_V, the item
//                     records; after the per-chunk barrier
//                     warp 4 issues the PV MMAs, warp 5 the QK MMAs and warps
//                     6-7 (the loaders) refill the ring, popping the next items
//                     from the queue well ahead of use.
// One CTA barrier per chunk publishes the TMEM / shared operands; QK(k+1)
// (incl. the key zero term A_ones B_Z) and PV(k) are then issued together and
// complete on separate mbarriers.  Item boundaries do not drain the pipeline:
// the per-item state resets in the token / channel roles, and an item's record
// is published with a release add on its unit's arrival counter.
// Returns the first non-quantized item popped (or >= nitems).
template <int NG>
__device__ int run_quant_stream(const DecArgs& a, int nq, TcSmem& sm, uint32_t tb, uint32_t& qk_ph,
                                uint32_t& pv_ph) {
  const kvlc_cache& c = a.c;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool tok = warp < 4, loader = warp >= 6;
  const int row = tid & 127;
  const uint32_t lane_addr = tb + ((uint32_t)(32 * (warp & 3)) << 16);
  const float f4 = __int_as_float((127 - 2 * ((row >> 1) & 3)) << 23);  // 4^-p(row)

  // ---- loaders (warps 6-7): stream chunk L into ring stage L % NSTAGE.  The item
  // being loaded lives in (uniform) registers; the queue is popped only when it
  // is exhausted, by one lane, published to the other loader lanes through
  // shared memory and named barrier 2.
  auto item_n = [&](int unit, int split) {
    const int b = unit / c.Hkv;
    const int n_ch = min(c.n_chunks[b], a.chunk_hi);
    const int lo = a.chunk_lo + split * a.cpc;
    return max(0, min(n_ch, lo + a.cpc) - lo);
  };
  int ld_j = 0, ld_n = 0, ld_L = 0;
  bool ld_end = false;
  size_t ld_cb = 0;
  uint32_t ticket = loader && tid == 192 ? atomicAdd(a.queue, 1u) : 0u;  // next queue ticket, fetched ahead
  auto loader_step = [&]() {
    while (!ld_end && ld_j == ld_n) {
      if (tid == 192) {
        const int x = (int)ticket;
        if (x < nq) ticket = atomicAdd(a.queue, 1u);  // the following one, in flight meanwhile
        sm.empty_unit = -1;
        if (x < nq) {
          const int unit = x / a.nsq, split = x % a.nsq, n = item_n(unit, split);
          if (n > 0) {
            sm.items[sm.n_items & (IFIFO - 1)] = QItem{unit, split, n};
            sm.n_items = sm.n_items + 1;
          } else {
            sm.empty_unit = unit;
            sm.empty_split = split;
          }
        } else {
          sm.next = x;
          sm.end = ld_L;
        }
      }
      lbar_sync();
      if (sm.end >= 0) {
        ld_end = true;
      } else if (sm.empty_unit >= 0) {  // an item without chunks (short sequence): empty record
        const int eu = sm.empty_unit;
        float* rec = a.rec + ((size_t)eu * a.nrec + sm.empty_split) * NG * REC;
        for (int i = tid - 192; i < NG * REC; i += 64) {
          const int kk = i % REC;
          rec[i] = (kk == 0 || kk == 2) ? -INFINITY : 0.f;
        }
        lbar_sync();
        if (tid == 192) red_release_add(a.done + eu, 1u);
      } else {
        const int slot = (sm.n_items - 1) & (IFIFO - 1);
        const QItem q = sm.items[slot];
        ld_n = q.n;
        ld_j = 0;
        ld_cb = (size_t)q.unit * c.max_chunks + a.chunk_lo + (size_t)q.split * a.cpc;
        // the item's NG query vectors -> sm.qv[slot] (16 B pieces), completes with this chunk's group
        const int b = q.unit / c.Hkv, kvh = q.unit % c.Hkv;
        const uint16_t* qsrc = a.q + ((size_t)b * c.Hq + (size_t)kvh * NG) * D;
        for (int i = tid - 192; i < NG * 16; i += 64)
          tc::cp_async16(&sm.qv[slot][i >> 4][8 * (i & 15)], qsrc + (i >> 4) * D + 8 * (i & 15));
      }
      lbar_sync();  // scratch fields are rewritten by the next pop
    }
    if (!ld_end) {
      ChunkStage& S = sm.stage[ld_L % NSTAGE];
      const size_t cb = ld_cb + ld_j;
      const uint4* kc = reinterpret_cast<const uint4*>(c.kcodes + cb * 1024);
      const uint4* vc = reinterpret_cast<const uint4*>(c.vcodes + cb * 1024);
      const int i0 = tid - 192;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) tc::cp_async16(&S.kc[i0 + 64 * jj], kc + i0 + 64 * jj);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) tc::cp_async16(&S.vc[i0 + 64 * jj], vc + i0 + 64 * jj);
      {
        const int which = i0 >> 4, part = i0 & 15;  // 64 pieces: ks, kz, vs, vz
        const uint16_t* src = (which == 0 ? c.kscale : which == 1 ? c.kzero : which == 2 ? c.vscale : c.vzero) + cb * D;
        uint16_t* dst = which == 0 ? S.ks : which == 1 ? S.kz : which == 2 ? S.vs : S.vz;
        tc::cp_async16(dst + 8 * part, src + 8 * part);
      }
      ++ld_j;
      ++ld_L;
      if (tid == 192) sm.loaded = ld_L;
    }
    tc::cp_commit();
  };

  if (tid == 0) {
    sm.n_items = 0;
    sm.loaded = 0;
    sm.end = -1;
    sm.next = 0x7fffffff;
  }
  for (int i = tid; i < 256; i += QTHREADS) {  // columns beyond the heads stay zero
    sm.bqk[0][i] = make_uint4(0u, 0u, 0u, 0u);
    sm.bqk[1][i] = make_uint4(0u, 0u, 0u, 0u);
    sm.bz[0][i] = make_uint4(0u, 0u, 0u, 0u);
    sm.bz[1][i] = make_uint4(0u, 0u, 0u, 0u);
    sm.bpv[0][i] = make_uint4(0u, 0u, 0u, 0u);
    sm.bpv[1][i] = make_uint4(0u, 0u, 0u, 0u);
  }
  {
    uint32_t ones[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ones[j] = 0x00010001u;  // fp16 2^-24 pairs
    if (tok) tc::tmem_st8(lane_addr + COL_ONES, ones);
  }
  __syncthreads();
  if (loader) {
#pragma unroll 1
    for (int s = 0; s < NSTAGE; ++s) loader_step();
    tc::cp_wait<NSTAGE - 2>();  // chunks 0, 1
  }
  tc::wait_st();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  int L = sm.loaded;
  if (L == 0) return sm.next;  // no quantized work left

  // token role: q factors (of channel `row`) of the item whose B_QK / B_Z rows are
  // being built (b_it), and the prefetched raw q of the following item (pre_it)
  float qf[NG], qz[NG];
  int b_it = 0;
  auto q_load = [&](int it, float* dst) {  // staged by the loaders with the item's first chunk
#pragma unroll
    for (int h = 0; h < NG; ++h) dst[h] = bf2f(sm.qv[it & (IFIFO - 1)][h][row]);
  };
  auto q_set = [&](const float* qv) {
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      qf[h] = qv[h] * (C0 * QK_SCALE) * f4;
      qz[h] = qv[h] * (C0 * QK_SCALE);
    }
  };
  auto build_bqk = [&](int k) {  // token role: B_QK / B_Z row `row` of stream chunk k
    const ChunkStage& S = sm.stage[k % NSTAGE];
    const float s = h2f(S.ks[row]), z = h2f(S.kz[row]);
    float x[NG], y[NG];
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      x[h] = qf[h] * s;
      y[h] = qz[h] * z;
    }
    write_brow<NG>(sm.bqk[k & 1], row, x);
    write_brow<NG>(sm.bz[k & 1], row, y);
  };
  auto issue_qk = [&](int k) {  // warp 5
    tc::mma16_qk_commit_w(tb + COL_DQK, tb + COL_AK + 64u * (uint32_t)(k & 1), tc::bdesc(tc::smem_u32(sm.bqk[k & 1])),
                          tb + COL_ONES, tc::bdesc(tc::smem_u32(sm.bz[k & 1])), &sm.mqk);
  };
  auto issue_pv = [&](int k) {  // warp 4
    tc::mma8_commit_w(tb + COL_DPV, tb + COL_AV, tc::bdesc(tc::smem_u32(sm.bpv[k & 1])), &sm.mpv);
  };

  // prologue: operands of chunk 0, QK(0)
  if (tok) {
    float q0[NG];
    q_load(0, q0);
    q_set(q0);
    expand_row(sm.stage[0].kc, row, lane_addr + COL_AK);
    build_bqk(0);
  } else {
    expand_row(sm.stage[0].vc, row, lane_addr + COL_AV);
  }
  tc::wait_st();
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 5) {
    tc::fence_after_sync();
    issue_qk(0);
  }

  // token role: reference point o (log2 units), l, sum p z_v, true max; channel role: numerator acc in frame oc
  float o[NG], l[NG], zs[NG], mt[NG], acc[NG], oc[NG];
  auto reset_tok = [&]() {
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      o[h] = -INFINITY;
      l[h] = 0.f;
      zs[h] = 0.f;
      mt[h] = -INFINITY;
    }
  };
  auto reset_chn = [&]() {
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      acc[h] = 0.f;
      oc[h] = -INFINITY;
    }
  };
  reset_tok();
  reset_chn();
  // channel role: PV of stream chunk k (frame ob[k & 1]) -> acc; if k ends its item, publish the record
  int pend_unit = -1, pend_k = 0;  // tid 224: an item record written at chunk pend_k, not yet released
  auto drain_pv = [&](int k, int it, bool last) {
    uint32_t dp[16];
    ld_d<NG>(lane_addr + COL_DPV, dp);
    tc::wait_ld();
    float d[NG];
    sum_d<NG>(dp, d);
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      const float on = sm.ob[k & 1][h];
      if (on != oc[h]) {  // warp-uniform; rare after an item's first chunk
        acc[h] *= oc[h] == -INFINITY ? 0.f : exp2f(oc[h] - on);
        oc[h] = on;
      }
      acc[h] = fmaf(d[h], 16777216.f, acc[h]);
    }
    if (last) {
      const QItem q = sm.items[it & (IFIFO - 1)];
      float* rec = a.rec + ((size_t)q.unit * a.nrec + q.split) * NG * REC;
      const float(*tr)[8][4] = sm.itred[it & 1];
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        const float Lh = (tr[0][h][0] + tr[1][h][0]) + (tr[2][h][0] + tr[3][h][0]);
        const float Z = (tr[0][h][1] + tr[1][h][1]) + (tr[2][h][1] + tr[3][h][1]);
        const float MT = fmaxf(fmaxf(tr[0][h][2], tr[1][h][2]), fmaxf(tr[2][h][2], tr[3][h][2]));
        float* r = rec + h * REC;
        if (row == 0) *reinterpret_cast<float4*>(r) = make_float4(oc[h], Lh, MT, 0.f);
        r[4 + row] = acc[h] + Z;  // numerator of channel row: sum_t p_t (s_t code_t + z_t), rotated basis
      }
      if (tid == 224) {  // released a few chunks later, when its writes are long complete (no fence stall)
        if (pend_unit >= 0) red_release_add(a.done + pend_unit, 1u);  // short items: release the older one now
        pend_unit = q.unit;
        pend_k = k;
      }
      reset_chn();
    }
  };

  int ci = 0, cj = 0;  // item (FIFO index) and chunk within it of stream chunk k
  int k = 0;
  for (; k < L; ++k) {
    const int n_ci = sm.items[ci & (IFIFO - 1)].n;
    const bool first = cj == 0, last = cj == n_ci - 1;
    const bool more = k + 1 < L;
    if (tok) {
      KVLC_STAMP(k, 0);
      // chunk k+1's K rows into the other A_K buffer, its B_QK / B_Z rows into the
      // other B buffers (their last reader QK(k-1) is complete)
      if (more) {
        expand_row(sm.stage[(k + 1) % NSTAGE].kc, row, lane_addr + COL_AK + 64u * (uint32_t)((k + 1) & 1));
        const int nb = last ? ci + 1 : ci;  // item of chunk k+1
        if (nb != b_it) {                   // a new item: its q (staged in shared memory)
          float qn[NG];
          q_load(nb, qn);
          q_set(qn);
          b_it = nb;
        }
        build_bqk(k + 1);
      }
      KVLC_STAMP(k, 1);
      tc::mbar_wait(&sm.mqk, (qk_ph + (uint32_t)k) & 1u);  // QK(k) complete
      tc::fence_after_sync();
      KVLC_STAMP(k, 2);
      float l2[NG];
      {
        uint32_t dq[16];
        ld_d<NG>(lane_addr + COL_DQK, dq);
        tc::wait_ld();
        sum_d<NG>(dq, l2);
      }
      if (first) reset_tok();
      bool ev = false;
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        l2[h] *= 16777216.f / QK_SCALE;  // logit incl. the key zero term, log2 units (C0 folded into q)
        ev |= l2[h] > o[h] + LAZY;
      }
      if (tbar_or(ev)) {  // move the reference point (item start, or a new maximum)
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          const float m = warp_max(l2[h]);
          if (lane == 0) sm.red[warp][h][0] = m;
        }
        tbar_sync();
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          const float m = fmaxf(fmaxf(sm.red[0][h][0], sm.red[1][h][0]), fmaxf(sm.red[2][h][0], sm.red[3][h][0]));
          const float on = fmaxf(o[h], m);
          const float f = o[h] == -INFINITY ? 0.f : exp2f(o[h] - on);
          l[h] *= f;
          zs[h] *= f;
          o[h] = on;
        }
        tbar_sync();  // red[] is reused
      }
      KVLC_STAMP(k, 3);
      const ChunkStage& S = sm.stage[k % NSTAGE];
      const float sv = h2f(S.vs[row]) * f4, zv = h2f(S.vz[row]);
      float pv[NG];
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        const float p = fast_exp2(l2[h] - o[h]);
        l[h] += p;
        zs[h] = fmaf(p, zv, zs[h]);
        mt[h] = fmaxf(mt[h], l2[h]);
        pv[h] = p * sv;
      }
      write_brow<NG>(sm.bpv[k & 1], row, pv);
      if (row < NG) sm.ob[k & 1][row] = o[row];
      if (last) {  // per-warp item totals for the channel role's record
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          const float ls = warp_sum(l[h]), zz = warp_sum(zs[h]), mm = warp_max(mt[h]);
          if (lane == 0) {
            sm.itred[ci & 1][warp][h][0] = ls;
            sm.itred[ci & 1][warp][h][1] = zz;
            sm.itred[ci & 1][warp][h][2] = mm;
          }
        }
      }
      KVLC_STAMP(k, 4);
    } else {
      KVLC_STAMP(k, 8);
      if (tid == 224 && pend_unit >= 0 && k >= pend_k + 3) {  // its writes are long complete: cheap fence
        red_release_add(a.done + pend_unit, 1u);
        pend_unit = -1;
      }
      if (k > 0) {
        tc::mbar_wait(&sm.mpv, (pv_ph + (uint32_t)(k - 1)) & 1u);  // PV(k-1) complete: D_PV and A_V are free
        tc::fence_after_sync();
        KVLC_STAMP(k, 9);
        // stream chunk k-1 ended its item iff chunk k starts one
        drain_pv(k - 1, first ? ci - 1 : ci, first);
        KVLC_STAMP(k, 10);
        expand_row(sm.stage[k % NSTAGE].vc, row, lane_addr + COL_AV);
      }
      KVLC_STAMP(k, 11);
    }
    if (loader) tc::cp_wait<NSTAGE - 3>();  // chunk k+2 landed; visible to all after the barrier
    tc::wait_st();
    tc::fence_proxy_async();
    tc::fence_before_sync();
    KVLC_STAMP_WARP(k);
    __syncthreads();
    KVLC_STAMP(k, tok ? 5 : 13);
    if (warp == 5) {
      tc::fence_after_sync();
      if (more) issue_qk(k + 1);
    } else if (warp == 4) {
      tc::fence_after_sync();
      issue_pv(k);
    } else if (loader) {
      loader_step();  // chunk k's stage is fully consumed
    }
    KVLC_STAMP(k, tok ? 6 : 14);
    if (last) {
      ++ci;
      cj = 0;
    } else {
      ++cj;
    }
    // sm.loaded may be bumped concurrently by the loaders of this iteration; either
    // value gives the same answer to "chunk k+2 exists" (the ring runs NSTAGE >= 3 ahead,
    // and a finished stream no longer changes it)
    L = sm.loaded;
  }
  if (!tok) {  // last PV and record
    tc::mbar_wait(&sm.mpv, (pv_ph + (uint32_t)(k - 1)) & 1u);
    tc::fence_after_sync();
    drain_pv(k - 1, ci - 1, true);
    cbar_sync();  // every channel thread has written the last record
    if (tid == 224) red_release_add(a.done + pend_unit, 1u);
  }
  if (loader) tc::cp_wait<0>();
  tc::fence_before_sync();
  __syncthreads();
  qk_ph += (uint32_t)k;
  pv_ph += (uint32_t)k;
  return sm.next;
}
