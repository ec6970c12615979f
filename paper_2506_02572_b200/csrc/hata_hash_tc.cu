// Prefill key hash on the tensor cores (bf16): codes = pack(sign(K_tile . W_g)).
//
// PAPER: Alg. 1 lines 2-5 with HashEncode = Alg. 2:
// Sign(MatMul(K, W_H)) -> BitPack, done once per cached key at prefill
// ("<1% of total computation").
//
// A K tile = 128 tokens of one (b, g) x all rbits output bits; 8 warps, warp
// w owns tokens [16w, 16w+16).  K tiles and W_g are staged in smem (padded rows, so
// the ldmatrix fragments are bank-conflict free); every 16 x 8 output tile is
// one chain of D/16 mma.sync m16n8k16 (bf16 products are exact, fp32
// accumulation, R13), four chains per code word; each lane packs the sign bits
// of its accumulator fragments into its 2 bits per n-tile of the LSB-first
// uint32 word and the 4 lanes of a row OR-reduce by shuffles (R6, R7).
//
// This is the legacy-MMA (HMMA) path: at rbits = 128 the projection needs
// 128 flop per K byte, so HMMA (~0.58 PFLOP/s on this part) rather than HBM
// bounds it; a tcgen05/TMEM version is the next step.
#include "hata_internal.h"
#include "hata_common.cuh"

namespace hata {

constexpr int HK_MT = 2;                     // 16-token m-tiles per warp (share every W_g fragment)
constexpr int HK_THREADS = 128;
constexpr int HK_TOK = HK_THREADS / 32 * 16 * HK_MT;   // tokens per CTA tile (128)

// Persistent CTAs: CTA (x, u) hashes token tiles x, x + nx, x + 2 nx, ... of
// unit u = (b, g); W_g is staged once, K tiles are double-buffered with
// cp.async (the next tile streams in while the current one is on the MMAs).
template <int RB>                             // rbits
__global__ void __launch_bounds__(HK_THREADS) hash_keys_mma_kernel(const HashKeysParams p) {
  constexpr int D = 128;
  constexpr int W = RB / 32;
  constexpr int XROW = D * 2 + 16;            // padded smem row of the K tile (bytes)
  constexpr int WROW = RB * 2 + 16;           // padded smem row of W_g (bytes)
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* ws = sm;                           // [D][WROW]
  uint8_t* xs0 = sm + D * WROW;               // 2 x [HK_TOK][XROW]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int bg = blockIdx.y, b = bg / p.Hkv, g = bg % p.Hkv;
  const int ntiles = (int)((p.n + HK_TOK - 1) / HK_TOK);
  const __nv_bfloat16* Kb = reinterpret_cast<const __nv_bfloat16*>(p.K) + (int64_t)b * p.kv_sb + (int64_t)g * p.kv_sh;
  const __nv_bfloat16* Wg = reinterpret_cast<const __nv_bfloat16*>(p.Wh) + (int64_t)g * D * RB;
  uint32_t* cb = p.codes + (int64_t)b * p.c_sb + (int64_t)g * p.c_sh;
  constexpr int XCH = D * 2 / 16, WCH = RB * 2 / 16;

  auto stage_k = [&](int tile, uint8_t* xs) {   // K rows past the end are zero
    const int64_t tbase = p.t0 + (int64_t)tile * HK_TOK;
    const int ntok = (int)min((int64_t)HK_TOK, p.t0 + p.n - tbase);
    for (int i = tid; i < HK_TOK * XCH; i += HK_THREADS) {
      const int r = i / XCH, c = i % XCH;
      uint8_t* dst = xs + r * XROW + c * 16;
      if (r < ntok) cp_async16_g(dst, reinterpret_cast<const uint4*>(Kb + (tbase + r) * p.kv_st) + c);
      else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int i = tid; i < D * WCH; i += HK_THREADS) {
    const int r = i / WCH, c = i % WCH;
    *reinterpret_cast<uint4*>(ws + r * WROW + c * 16) = __ldg(reinterpret_cast<const uint4*>(Wg + (int64_t)r * RB) + c);
  }
  int buf = 0;
  if ((int)blockIdx.x < ntiles) stage_k(blockIdx.x, xs0);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int next = tile + gridDim.x;
    uint8_t* xs = xs0 + buf * (HK_TOK * XROW);
    if (next < ntiles) {
      stage_k(next, xs0 + (buf ^ 1) * (HK_TOK * XROW));
      asm volatile("cp.async.wait_group 1;" ::: "memory");       // current tile landed
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();

    constexpr int KS = D / 16;
    uint32_t a[HK_MT][KS][4];
#pragma unroll
    for (int mt = 0; mt < HK_MT; ++mt)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint8_t* ap = xs + ((warp * HK_MT + mt) * 16 + (lane & 15)) * XROW + ks * 32 + (lane >> 4) * 16;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a[mt][ks][0]), "=r"(a[mt][ks][1]), "=r"(a[mt][ks][2]), "=r"(a[mt][ks][3])
                     : "r"(smem_u32(ap)));
      }
    uint32_t wlo[HK_MT][W], whi[HK_MT][W];    // code words of rows gid and gid + 8 of each m-tile
#pragma unroll
    for (int w = 0; w < W; ++w) {
      // one code word = 4 output n-tiles: 4 x HK_MT independent accumulator chains
      float c[HK_MT][4][4];
#pragma unroll
      for (int mt = 0; mt < HK_MT; ++mt)
#pragma unroll
        for (int q = 0; q < 4; ++q) c[mt][q][0] = c[mt][q][1] = c[mt][q][2] = c[mt][q][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t b0, b1;
          ldsm_x2_trans(b0, b1, ws + (ks * 16 + (lane & 15)) * WROW + (4 * w + q) * 16);
#pragma unroll
          for (int mt = 0; mt < HK_MT; ++mt) mma_bf16_16816(c[mt][q], a[mt][ks], b0, b1);
        }
      // c0, c1: row gid, bits 8q + 2 tig (+1) of the word; c2, c3: row gid + 8.
      // Each lane sets its 2 bits per n-tile; the 4 lanes of a row OR-reduce.
#pragma unroll
      for (int mt = 0; mt < HK_MT; ++mt) {
        uint32_t lo = 0u, hi = 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          lo |= ((uint32_t)(c[mt][q][0] >= 0.f) | ((uint32_t)(c[mt][q][1] >= 0.f) << 1)) << (8 * q + 2 * tig);
          hi |= ((uint32_t)(c[mt][q][2] >= 0.f) | ((uint32_t)(c[mt][q][3] >= 0.f) << 1)) << (8 * q + 2 * tig);
        }
        lo |= __shfl_xor_sync(0xffffffffu, lo, 1);
        hi |= __shfl_xor_sync(0xffffffffu, hi, 1);
        lo |= __shfl_xor_sync(0xffffffffu, lo, 2);
        hi |= __shfl_xor_sync(0xffffffffu, hi, 2);
        wlo[mt][w] = lo;
        whi[mt][w] = hi;
      }
    }
    if (tig == 0) {
      const int64_t tbase = p.t0 + (int64_t)tile * HK_TOK;
      const int ntok = (int)min((int64_t)HK_TOK, p.t0 + p.n - tbase);
#pragma unroll
      for (int mt = 0; mt < HK_MT; ++mt) {
        const int r0 = (warp * HK_MT + mt) * 16 + gid, r1 = r0 + 8;
        if (r0 < ntok) {
#pragma unroll
          for (int w = 0; w < W; ++w) cb[(tbase + r0) * W + w] = wlo[mt][w];
        }
        if (r1 < ntok) {
#pragma unroll
          for (int w = 0; w < W; ++w) cb[(tbase + r1) * W + w] = whi[mt][w];
        }
      }
    }
    __syncthreads();                          // this buffer is refilled two tiles on
    buf ^= 1;
  }
  // codes visible GPU-wide before a dependent decode launch (which streams
  // code rows before its griddepcontrol.wait) may start: every writer
  // fences, the CTA syncs, then it triggers
  __threadfence();
  __syncthreads();
  griddep_launch_dependents();
}

template <int RB>
static cudaError_t launch_rb(const HashKeysParams& p, cudaStream_t s) {
  const size_t smem = (size_t)128 * (RB * 2 + 16) + 2 * (size_t)HK_TOK * (128 * 2 + 16);
  cudaError_t e = cudaFuncSetAttribute(hash_keys_mma_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int units = p.B * p.Hkv;
  const int ntiles = (int)((p.n + HK_TOK - 1) / HK_TOK);
  int per_sm = (int)(227 * 1024 / smem);
  if (per_sm < 1) per_sm = 1;
  int nx = (device_sm_count() * per_sm + units - 1) / units;   // CTAs per unit: fill the chip once
  if (nx > ntiles) nx = ntiles;
  if (nx < 1) nx = 1;
  hash_keys_mma_kernel<RB><<<dim3(nx, units), HK_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

// bf16, d = 128: rbits in {32, 64, 128, 256}; anything else -> not supported
// (the caller falls back to the CUDA-core kernel).
cudaError_t launch_hash_keys_tc(const HashKeysParams& p, cudaStream_t s) {
  if (p.d != 128 || p.n <= 0) return p.n <= 0 ? cudaSuccess : cudaErrorNotSupported;
  switch (p.rbits) {
    case 32: return launch_rb<32>(p, s);
    case 64: return launch_rb<64>(p, s);
    case 128: return launch_rb<128>(p, s);
    case 256: return launch_rb<256>(p, s);
  }
  return cudaErrorNotSupported;
}

}  // namespace hata
