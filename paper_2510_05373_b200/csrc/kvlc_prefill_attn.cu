// Corrected causal prefill attention on the tensor cores.
//
// Reference: corrected_attention_quadratic / corrected_attention_recurrent
// (attention.py:99-155) -- both return, for every query t,
//     out_t = sum_{i<=t} (e^{s_ti} + f_ti) v_i  /  sum_{i<=t} (e^{s_ti} + f_ti),
//     s_ti = q_t . k_i / sqrt(d),   f_ti = phi_q(q_t) . phi_k(k_err_i)
// (raw, unshifted exponentials; f = 0 without an adapter).  The float64 reference-
// semantics kernel is kvlc_ref_attention; this is the fast path for many heads and
// long prefixes, flash-attention style: one CTA per (head, 64-query block), key
// blocks of 64 streamed through shared memory, mma.sync m16n8k16 with fp32
// accumulation; q, k, v as fp16 hi / lo pairs (3 passes: hi.hi, hi.lo, lo.hi),
// phi_q . phi_k in one fp16 pass (entries in (0, 1), 256-term dot products).
// The running frame is the decode's consistent-correction rule (attention.py:
// 190-194): exponentials are shifted by M+ = max(0, running max), the correction
// term scaled by 2^-M+ with them, so neither overflows (the reference's fp64 raw
// exponentials) and an all-negative prefix keeps the correction at full weight.
#include "kvlc_common.cuh"

#include <cuda_fp16.h>

namespace kvlc {
namespace {

constexpr int PD = 128;        // head dim
constexpr int PR = 256;        // adapter rank (phi dim)
constexpr int QB = 64;         // queries per CTA (4 warps x 16 rows)
constexpr int KB = 64;         // keys per block
constexpr int LD = PD + 8;     // fp16 row stride of the q / k / v tiles (272 B: conflict-free ldmatrix)
constexpr int LDP = PR + 8;    // row stride of the phi tiles
constexpr int PA_THREADS = 128;

struct PaSmem {
  __half qh[QB * LD], ql[QB * LD], pq[QB * LDP];
  __half kh[KB * LD], kl[KB * LD], vh[KB * LD], vl[KB * LD], pk[KB * LDP];
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t (&r)[2], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n"
               : "=r"(r[0]), "=r"(r[1]) : "r"(su32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float x, float y) {
  __half2 h = __floats2half2_rn(x, y);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst)), "l"(src) : "memory");
}

// fp32 -> fp16 hi / lo images: q pre-scaled by log2(e) / sqrt(d) (scores in log2 units).
__global__ void pa_prep_kernel(const float* __restrict__ x, int64_t count, float scale, __half* __restrict__ hi,
                               __half* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i] * scale;
    const __half h = __float2half_rn(v);
    hi[i] = h;
    if (lo) lo[i] = __float2half_rn(v - __half2float(h));
  }
}

// A [rows][cols] tile (fp16, global row stride gcols) into shared memory (row stride ld);
// rows past n are zero.
__device__ __forceinline__ void load_tile(__half* dst, const __half* src, int row0, int n, int cols, int ld) {
  const int per_row = cols / 8;  // 16-B pieces
  for (int i = threadIdx.x; i < 64 * per_row; i += PA_THREADS) {
    const int r = i / per_row, c8 = (i % per_row) * 8;
    __half* d = dst + r * ld + c8;
    if (row0 + r < n)
      cp16(d, src + (size_t)(row0 + r) * cols + c8);
    else
      *reinterpret_cast<uint4*>(d) = make_uint4(0u, 0u, 0u, 0u);
  }
}

template <bool ADAPT>
__global__ void __launch_bounds__(PA_THREADS, 1)
    pa_kernel(const __half* __restrict__ qh, const __half* __restrict__ ql, const __half* __restrict__ kh,
              const __half* __restrict__ kl, const __half* __restrict__ vh, const __half* __restrict__ vl,
              const __half* __restrict__ pq, const __half* __restrict__ pk, int64_t n, float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char pa_raw[];
  PaSmem& sm = *reinterpret_cast<PaSmem*>(pa_raw);
  const int head = blockIdx.y, qb = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const size_t hoff = (size_t)head * n;
  const int q0 = qb * QB;
  load_tile(sm.qh, qh + hoff * PD, q0, (int)n, PD, LD);
  load_tile(sm.ql, ql + hoff * PD, q0, (int)n, PD, LD);
  if (ADAPT) load_tile(sm.pq, pq + hoff * PR, q0, (int)n, PR, LDP);

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY};  // running max of the scores (log2 units)
  float lrow[2] = {0.f, 0.f};              // this lane's partial row sums in the frame 2^-M+
  const int row_a = q0 + 16 * warp + g, row_b = row_a + 8;
  // ldmatrix source rows of this lane: A tiles (16 rows x 16 cols), B tiles (8 rows x 16 cols)
  const int a_r = 16 * warp + (lane & 15), a_c = (lane >> 4) * 8;
  const int b_r = lane & 7, b_c = ((lane >> 3) & 1) * 8;

  for (int kb = 0; kb <= qb; ++kb) {
    const int k0 = kb * KB;
    __syncthreads();  // the previous block's tiles are consumed
    load_tile(sm.kh, kh + hoff * PD, k0, (int)n, PD, LD);
    load_tile(sm.kl, kl + hoff * PD, k0, (int)n, PD, LD);
    load_tile(sm.vh, vh + hoff * PD, k0, (int)n, PD, LD);
    load_tile(sm.vl, vl + hoff * PD, k0, (int)n, PD, LD);
    if (ADAPT) load_tile(sm.pk, pk + hoff * PR, k0, (int)n, PR, LDP);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();

    // ---- S = q k^T (log2 units), 3 passes ----
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < PD / 16; ++ks) {
      uint32_t ah[4], al[4];
      ldsm_x4(ah, sm.qh + a_r * LD + 16 * ks + a_c);
      ldsm_x4(al, sm.ql + a_r * LD + 16 * ks + a_c);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        uint32_t bh[2], bl[2];
        ldsm_x2(bh, sm.kh + (8 * nt + b_r) * LD + 16 * ks + b_c);
        ldsm_x2(bl, sm.kl + (8 * nt + b_r) * LD + 16 * ks + b_c);
        mma16816(s[nt], ah, bh[0], bh[1]);
        mma16816(s[nt], ah, bl[0], bl[1]);
        mma16816(s[nt], al, bh[0], bh[1]);
      }
    }
    // ---- f = phi_q phi_k^T, one pass ----
    float f[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i][0] = f[i][1] = f[i][2] = f[i][3] = 0.f;
    if (ADAPT) {
#pragma unroll 4
      for (int ks = 0; ks < PR / 16; ++ks) {
        uint32_t a[4];
        ldsm_x4(a, sm.pq + a_r * LDP + 16 * ks + a_c);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          uint32_t b[2];
          ldsm_x2(b, sm.pk + (8 * nt + b_r) * LDP + 16 * ks + b_c);
          mma16816(f[nt], a, b[0], b[1]);
        }
      }
    }
    // ---- causal mask, running max, weights w = 2^(s - M+) + f 2^-M+ ----
    float bmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + 8 * nt + 2 * t + (e & 1), row = e < 2 ? row_a : row_b;
        const bool ok = key <= row && key < n;
        s[nt][e] = ok ? s[nt][e] : -INFINITY;
        if (!ok) f[nt][e] = 0.f;
        bmax[e >> 1] = fmaxf(bmax[e >> 1], s[nt][e]);
      }
    float mp[2], sc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float m = bmax[r];
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
      const float mold = fmaxf(mrow[r], 0.f);
      mrow[r] = fmaxf(mrow[r], m);
      mp[r] = fmaxf(mrow[r], 0.f);            // M+ = max(0, running max)
      sc[r] = exp2f(mold - mp[r]);            // frame change of the accumulated rows
      lrow[r] *= sc[r];
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= sc[0];
      o[i][1] *= sc[0];
      o[i][2] *= sc[1];
      o[i][3] *= sc[1];
    }
    const float cf[2] = {exp2f(-mp[0]), exp2f(-mp[1])};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const float w = exp2f(s[nt][e] - mp[r]) + f[nt][e] * cf[r];
        s[nt][e] = w;
        lrow[r] += w;
      }
    // ---- o += w v (w as A fragments: hi / lo; v hi / lo; 3 passes) ----
#pragma unroll
    for (int kk = 0; kk < KB / 16; ++kk) {
      uint32_t wh[4], wl[4];
      const float* w0 = s[2 * kk];
      const float* w1 = s[2 * kk + 1];
      const float wv[8] = {w0[0], w0[1], w0[2], w0[3], w1[0], w1[1], w1[2], w1[3]};
      float hv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) hv[i] = __half2float(__float2half_rn(wv[i]));
      wh[0] = pack_h2(hv[0], hv[1]);
      wh[1] = pack_h2(hv[2], hv[3]);
      wh[2] = pack_h2(hv[4], hv[5]);
      wh[3] = pack_h2(hv[6], hv[7]);
      wl[0] = pack_h2(wv[0] - hv[0], wv[1] - hv[1]);
      wl[1] = pack_h2(wv[2] - hv[2], wv[3] - hv[3]);
      wl[2] = pack_h2(wv[4] - hv[4], wv[5] - hv[5]);
      wl[3] = pack_h2(wv[6] - hv[6], wv[7] - hv[7]);
      const int vr = 16 * kk + (lane & 15);  // ldmatrix.trans rows = keys
#pragma unroll
      for (int nv = 0; nv < 16; ++nv) {
        uint32_t bh[2], bl[2];
        ldsm_x2_t(bh, sm.vh + vr * LD + 8 * nv);
        ldsm_x2_t(bl, sm.vl + vr * LD + 8 * nv);
        mma16816(o[nv], wh, bh[0], bh[1]);
        mma16816(o[nv], wh, bl[0], bl[1]);
        mma16816(o[nv], wl, bh[0], bh[1]);
      }
    }
  }
  // ---- divide, store fp32 rows ----
  float lsum[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float l = lrow[r];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    lsum[r] = l;
  }
#pragma unroll
  for (int nv = 0; nv < 16; ++nv) {
    const int col = 8 * nv + 2 * t;
    if (row_a < n)
      *reinterpret_cast<float2*>(out + (hoff + row_a) * PD + col) = make_float2(o[nv][0] / lsum[0], o[nv][1] / lsum[0]);
    if (row_b < n)
      *reinterpret_cast<float2*>(out + (hoff + row_b) * PD + col) = make_float2(o[nv][2] / lsum[1], o[nv][3] / lsum[1]);
  }
}

}  // namespace
}  // namespace kvlc

using namespace kvlc;

extern "C" {

size_t kvlc_corrected_attention_workspace(int64_t n, int heads, int rank) {
  const size_t e = (size_t)heads * n;
  return align_up(6 * e * PD * sizeof(__half)) + (rank ? align_up(2 * e * PR * sizeof(__half)) : 0);
}

int kvlc_corrected_attention(const float* q, const float* k, const float* v, const float* phq, const float* phk,
                             int64_t n, int heads, int rank, float* out, void* ws, size_t ws_bytes, void* stream) {
  KVLC_NEED_DEVICE();
  KVLC_REQUIRE(q && k && v && out && n >= 1 && heads >= 1, "bad corrected-attention arguments");
  KVLC_REQUIRE(rank == 0 || rank == PR, "adapter rank %d (the fast path takes %d or none)", rank, PR);
  KVLC_REQUIRE(!rank || (phq && phk), "rank %d needs phi_q / phi_k", rank);
  KVLC_REQUIRE(ws && ws_bytes >= kvlc_corrected_attention_workspace(n, heads, rank),
               "corrected-attention workspace too small (%zu bytes)", ws_bytes);
  cudaStream_t s = as_stream(stream);
  const size_t e = (size_t)heads * n;
  __half* base = static_cast<__half*>(ws);
  __half *qh = base, *ql = qh + e * PD, *kh = ql + e * PD, *kl = kh + e * PD, *vh = kl + e * PD, *vl = vh + e * PD;
  __half* pq = reinterpret_cast<__half*>(reinterpret_cast<char*>(ws) + align_up(6 * e * PD * sizeof(__half)));
  __half* pk = pq + e * PR;
  const int grid = 148 * 8;
  const float qscale = 1.4426950408889634f / sqrtf((float)PD);  // scores in log2 units
  pa_prep_kernel<<<grid, 256, 0, s>>>(q, (int64_t)(e * PD), qscale, qh, ql);
  pa_prep_kernel<<<grid, 256, 0, s>>>(k, (int64_t)(e * PD), 1.f, kh, kl);
  pa_prep_kernel<<<grid, 256, 0, s>>>(v, (int64_t)(e * PD), 1.f, vh, vl);
  if (rank) {
    pa_prep_kernel<<<grid, 256, 0, s>>>(phq, (int64_t)(e * PR), 1.f, pq, nullptr);
    pa_prep_kernel<<<grid, 256, 0, s>>>(phk, (int64_t)(e * PR), 1.f, pk, nullptr);
  }
  const dim3 g((unsigned)((n + QB - 1) / QB), (unsigned)heads);
  const size_t smem = sizeof(PaSmem);
  if (rank) {
    KVLC_CUDA(cudaFuncSetAttribute(pa_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pa_kernel<true><<<g, PA_THREADS, smem, s>>>(qh, ql, kh, kl, vh, vl, pq, pk, n, out);
  } else {
    KVLC_CUDA(cudaFuncSetAttribute(pa_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pa_kernel<false><<<g, PA_THREADS, smem, s>>>(qh, ql, kh, kl, vh, vl, pq, pk, n, out);
  }
  return check_launch("corrected_attention");
}

}  // extern "C"
