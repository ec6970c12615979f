// Sequence-sharded decode phases 2-4: global merge of
// the ranks' top-k' candidates, partial attention over own rows, and the
// rank-ordered flash-decoding combine.  Phase 1 is the decode kernel in
// candidate mode (hata_decode.cuh).
//
// PAPER: Alg. 3 lines 12-17 distributed over token ranges; the
// paper itself is single-GPU, so the split is this build's.
#include "hata_internal.h"
#include "hata_common.cuh"

namespace hata {



// One CTA per (b, g).  Candidates are visited rank-major then in list order,
// which is ascending global token order, so the lowest-index tie rule (R8)
// is a prefix quota exactly as in the single-GPU select.
__global__ void __launch_bounds__(256) shard_select_kernel(SelectParams p) {
  extern __shared__ __align__(16) int32_t ssm[];
  const int nbins = p.G * p.rbits + 1;
  int32_t* hist = ssm;                     // [nbins]
  int32_t* sbuf = ssm + nbins;             // [k] selected global indices, ascending
  int32_t* misc = sbuf + p.k;              // [64]
  const int bg = blockIdx.x, b = bg / p.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = blockDim.x / 32;
  const int64_t ntot = p.n_total[b];
  const int kp = (int)(ntot < p.k ? ntot : p.k);
  const int E = p.P * p.k;                 // candidate entries
  auto entry = [&](int e, int& D, int& idx) {
    const int rr = e / p.k, i = e % p.k;
    const int64_t off = (int64_t)rr * p.rank_stride + (int64_t)bg * p.k + i;
    idx = p.all_idx[off];
    D = idx >= 0 ? p.all_D[off] : 0x7fffffff;
  };
  for (int i = tid; i < nbins; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) {
    int D, idx;
    entry(e, D, idx);
    if (idx >= 0) atomicAdd(&hist[D], 1);
  }
  __syncthreads();
  if (warp == 0) {
    int before = 0, T = -1, below = 0;
    for (int i0 = 0; i0 < nbins && T < 0; i0 += 32) {
      const int v = i0 + lane < nbins ? hist[i0 + lane] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const uint32_t mm = __ballot_sync(0xffffffffu, before + inc >= kp && i0 + lane < nbins);
      if (mm) {
        const int l = __ffs(mm) - 1;
        T = i0 + l;
        below = __shfl_sync(0xffffffffu, before + inc - v, l);
      } else {
        before += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    if (kp <= 0) { T = -1; below = 0; }
    if (lane == 0) { misc[0] = T; misc[1] = kp - below; }
  }
  __syncthreads();
  const int T = misc[0], quota = misc[1];
  const int seg = ((E + NW - 1) / NW + 31) & ~31;
  const int s0 = min(E, warp * seg), s1 = min(E, s0 + seg);
  int lt_w = 0, ti_w = 0;
  for (int j0 = s0; j0 < s1; j0 += 32) {
    int D = 0x7fffffff, idx = -1;
    if (j0 + lane < s1) entry(j0 + lane, D, idx);
    lt_w += __popc(__ballot_sync(0xffffffffu, D < T));
    ti_w += __popc(__ballot_sync(0xffffffffu, D == T));
  }
  int* wcnt = misc + 8;
  if (lane == 0) { wcnt[2 * warp] = lt_w; wcnt[2 * warp + 1] = ti_w; }
  __syncthreads();
  int lt_b = 0, ti_b = 0;
  for (int w = 0; w < warp; ++w) { lt_b += wcnt[2 * w]; ti_b += wcnt[2 * w + 1]; }
  const int Gr = p.G * p.rbits;
  for (int j0 = s0; j0 < s1; j0 += 32) {
    int D = 0x7fffffff, idx = -1;
    if (j0 + lane < s1) entry(j0 + lane, D, idx);
    const uint32_t lm = __ballot_sync(0xffffffffu, D < T);
    const uint32_t tm = __ballot_sync(0xffffffffu, D == T);
    const uint32_t below_me = (1u << lane) - 1u;
    const int tr = ti_b + __popc(tm & below_me);
    if (D < T || (D == T && tr < quota)) {
      const int pos = lt_b + __popc(lm & below_me) + min(tr, quota);
      sbuf[pos] = idx;
      if (p.sel_idx) p.sel_idx[(int64_t)bg * p.k + pos] = idx;
      if (p.sel_score) p.sel_score[(int64_t)bg * p.k + pos] = Gr - 2 * D;
    }
    lt_b += __popc(lm);
    ti_b += __popc(tm);
  }
  __syncthreads();
  // own range [lo, hi) is a contiguous run of the ascending selection
  if (tid == 0) {
    int a = 0, z = kp;
    while (a < z) { int m = (a + z) / 2; if (sbuf[m] < p.lo) a = m + 1; else z = m; }
    int e = a, z2 = kp;
    while (e < z2) { int m = (e + z2) / 2; if (sbuf[m] < p.hi) e = m + 1; else z2 = m; }
    misc[2] = a; misc[3] = e;
    p.own_cnt[bg] = e - a;
  }
  __syncthreads();
  const int a = misc[2], e = misc[3];
  for (int i = tid; i < p.k; i += blockDim.x) {
    p.own_idx[(int64_t)bg * p.k + i] = (a + i < e) ? (int32_t)(sbuf[a + i] - p.lo) : -1;
    if (i >= kp) {
      if (p.sel_idx) p.sel_idx[(int64_t)bg * p.k + i] = -1;
      if (p.sel_score) p.sel_score[(int64_t)bg * p.k + i] = 0;
    }
  }
}

// Rank-ordered merge of P flash-decoding partials (m, l, acc[d]) per (b, h).
template <typename TO>
__global__ void shard_combine_kernel(const float* __restrict__ part, int P, int BH, int d, TO* out) {
  const int bh = blockIdx.x;
  const int stride = d + 2;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float M = -INFINITY;
    for (int r = 0; r < P; ++r) M = fmaxf(M, part[((int64_t)r * BH + bh) * stride]);
    float L = 0.f, A = 0.f;
    for (int r = 0; r < P; ++r) {
      const float* pr = part + ((int64_t)r * BH + bh) * stride;
      const float sc = (pr[0] == -INFINITY) ? 0.f : expf(pr[0] - M);
      L = fmaf(pr[1], sc, L);
      A = fmaf(pr[2 + e], sc, A);
    }
    const float o = L > 0.f ? A / L : 0.f;
    if constexpr (sizeof(TO) == 2) out[(int64_t)bh * d + e] = __float2bfloat16_rn(o);
    else out[(int64_t)bh * d + e] = o;
  }
}

cudaError_t launch_shard_select(const SelectParams& p, cudaStream_t s) {
  const size_t smem = ((size_t)(p.G * p.rbits + 1) + p.k + 64) * 4;
  cudaError_t e = cudaFuncSetAttribute(shard_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  shard_select_kernel<<<p.B * p.Hkv, 256, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_shard_combine(const float* part, int P, int B, int Hq, int d, void* out, int out_bf16,
                                 cudaStream_t s) {
  if (out_bf16)
    shard_combine_kernel<__nv_bfloat16><<<B * Hq, 128, 0, s>>>(part, P, B * Hq, d,
                                                                reinterpret_cast<__nv_bfloat16*>(out));
  else
    shard_combine_kernel<float><<<B * Hq, 128, 0, s>>>(part, P, B * Hq, d, reinterpret_cast<float*>(out));
  return cudaGetLastError();
}

}  // namespace hata
