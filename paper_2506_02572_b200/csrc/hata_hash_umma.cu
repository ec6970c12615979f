// Prefill key hash on the 5th-generation tensor cores (tcgen05 / TMEM / TMA):
// codes[t] = BitPack(Sign(K[t] . W_g)).
//
// PAPER: Alg. 1 lines 2-5 with HashEncode = Alg. 2:
// K_H <- BitPack(Sign(MatMul(K, W_H))), once per cached key at prefill
// ("<1% of total computation").  bf16 inputs, fp32 accumulation
// (R13), bit b = (p_b >= 0) (R6), LSB-first words (R7).
//
// One CTA = one (b, KV head) unit and a contiguous range of 128-token tiles:
//   warp 0   TMA producer: each K tile [128 tokens x 128] bf16 arrives as two
//            128-byte-swizzled [128 x 64] boxes (cp.async.bulk.tensor, one
//            tensor map over the K cache) into a 5-6 stage shared-memory ring
//            (the first stages stream in while W_g^T is staged);
//   warp 1   MMA issuer (one thread) + TMEM owner: D[128 x N] (fp32, TMEM) =
//            A[128 x 128] . B[128 x N] as 8 tcgen05.mma kind::f16 (K = 16
//            each), A = the K tile, B = W_g^T resident in shared memory
//            (K-major, swizzled once per CTA); two accumulators in TMEM so
//            the epilogue of tile i overlaps the MMAs of tile i + 1;
//   warps 2.. epilogue: 4 or 8 warps (two per TMEM lane quadrant when
//            rbits >= 64, each taking half of the columns); tcgen05.ld 32
//            columns per load, all loads in flight before one wait (one
//            TMEM lane = one token), 32 sign bits -> one code word, stores.
// N = rbits (32..256).  Synchronisation: mbarriers (TMA -> MMA full, MMA ->
// TMA empty via tcgen05.commit, MMA -> epilogue accumulator full via
// tcgen05.commit, epilogue -> MMA accumulator empty).
#include <cstring>
#include <cuda.h>                 // CUtensorMap (encoded through the runtime's driver entry point; no -lcuda)
#include "hata_internal.h"
#include "hata_common.cuh"

namespace hata {
namespace {

constexpr int UM_TOK = 128;                  // tokens per tile = UMMA M
// epilogue warps: 4 (one per TMEM lane quadrant) x EPI_SPLIT column groups
template <int N>
constexpr int epi_split() { return N >= 64 ? 2 : 1; }
template <int N, bool F = false>
constexpr int um_threads() { return 64 + 128 * epi_split<N>() + (F ? 32 : 0); }   // TMA, MMA, epilogue (+ store) warps
constexpr int UM_SLAB = UM_TOK * 128;        // one [128 rows x 64 bf16] swizzled box (16 KB)

// ---- tcgen05 / TMA primitives (inline PTX, sm_100a)
// Shared-memory matrix descriptor, K-major, SWIZZLE_128B: 128-byte rows, 8-row
// groups 1024 B apart (stride byte offset), leading byte offset unused.
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                    // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // layout: SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: D fp32, A and B bf16, both K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(UM_TOK >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// arrive on an mbarrier once every tcgen05 op issued so far by this thread completes
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// 32 lanes x 32 columns of 32-bit accumulators -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int N>
constexpr int tmem_cols() {                  // two accumulators, power of two >= 32
  return 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 2 * N <= 256 ? 256 : 512;
}
// bytes of one ring stage: the K tile (two swizzled slabs) [+ the V tile when
// the prefill write is fused]
template <bool F>
constexpr int stage_bytes() { return 2 * UM_SLAB * (F ? 2 : 1); }
// ring depth: as many stages as fit beside W_g^T (<= 6)
template <int N, bool F = false>
constexpr int um_stages() {
  return (227 * 1024 - 1024 - 2 * N * 128 - 256) / stage_bytes<F>() > 6 ? 6
                                                                        : (227 * 1024 - 1024 - 2 * N * 128 - 256) / stage_bytes<F>();
}
template <int N, bool F = false>
constexpr size_t umma_smem_bytes() {
  return 1024 + (size_t)2 * N * 128 + (size_t)um_stages<N, F>() * stage_bytes<F>() + 256;
}

// FUSED (NEXT-1, hata_prefill_write): the K tile comes from the new chunk
// (3-D maps {d, token, unit}), the same smem tile is also stored to the K
// cache and a V tile is carried through the stage to the V cache -- the keys
// are read from HBM once for both the cache write and the hash.
struct FusedMaps {
  CUtensorMap Kd, Vs, Vd;   // K cache (store), V chunk (load), V cache (store)
};

template <int N, bool FUSED>
__global__ void __launch_bounds__(um_threads<N, FUSED>(), 1)
    hash_keys_umma_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ FusedMaps fm,
                          const HashKeysParams p, int64_t row_sb, int64_t row_sh, int ntiles_unit, int tiles_per_cta) {
  constexpr int W = N / 32;
  constexpr int UM_THREADS = um_threads<N, FUSED>();
  constexpr int ES = epi_split<N>();
  constexpr int WE = W / ES;                 // code words per epilogue thread
  constexpr int UM_STAGES = um_stages<N, FUSED>();
  constexpr int SB = stage_bytes<FUSED>();
  constexpr int EPI_W0 = 2, EPI_W1 = 2 + 4 * ES;            // epilogue warps [EPI_W0, EPI_W1); store warp = EPI_W1
  constexpr uint32_t IDESC = idesc_bf16_f32(N);
  constexpr int BSLAB = N * 128;             // one [N x 64] swizzled slab of W_g^T
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* Bs = sm;                                        // W_g^T, 2 slabs
  uint8_t* As = sm + 2 * BSLAB;                            // ring: UM_STAGES x 2 slabs
  uint64_t* full = reinterpret_cast<uint64_t*>(As + UM_STAGES * SB);
  uint64_t* empty = full + UM_STAGES;
  uint64_t* tfull = empty + UM_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int u = blockIdx.y, b = u / p.Hkv, g = u % p.Hkv;
  const int tile0 = blockIdx.x * tiles_per_cta;
  const int my_tiles = max(0, min(ntiles_unit, tile0 + tiles_per_cta) - tile0);

  const int64_t row_unit = (int64_t)b * row_sb + (int64_t)g * row_sh;   // tensor-map row of (b, g, t = 0)
  auto produce = [&](int i) {                              // TMA: K (and V) tile i into stage i % UM_STAGES
    const int s = i % UM_STAGES;
    mbar_arrive_expect_tx(&full[s], SB);
    if constexpr (FUSED) {
      const int tsrc = (tile0 + i) * UM_TOK;                 // chunk row
      tma_load_3d(As + s * SB, &tmK, 0, tsrc, u, &full[s]);
      tma_load_3d(As + s * SB + UM_SLAB, &tmK, 64, tsrc, u, &full[s]);
      tma_load_3d(As + s * SB + 2 * UM_SLAB, &fm.Vs, 0, tsrc, u, &full[s]);
    } else {
      const int row = (int)(row_unit + p.t0 + (int64_t)(tile0 + i) * UM_TOK);
      tma_load_2d(As + s * SB, &tmK, 0, row, &full[s]);
      tma_load_2d(As + s * SB + UM_SLAB, &tmK, 64, row, &full[s]);
    }
  };
  if (tid == 0) {
    // a stage is free once its MMAs are done (tcgen05.commit) [and, fused,
    // once the store warp's TMA stores have read it]
    for (int s = 0; s < UM_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], FUSED ? 2 : 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4 * ES); }
    fence_mbar_init();
    // the first K tiles stream in while W_g^T is staged below
    for (int i = 0; i < UM_STAGES && i < my_tiles; ++i) produce(i);
  }
  if (warp == 1) {                                         // TMEM: two fp32 accumulators of N columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(tmem_cols<N>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // W_g^T into shared memory, K-major with the 128-byte swizzle (the layout
  // the MMA descriptor names): 16-byte chunk c of row n holds k = 8c .. 8c+7
  // of slab k / 64, stored at chunk c ^ (n % 8)
  {
    const uint16_t* Wg = reinterpret_cast<const uint16_t*>(p.Wh) + (int64_t)g * 128 * N;
    for (int i = tid; i < N * 16; i += UM_THREADS) {
      const int n = i % N, c16 = i / N;                    // consecutive threads: consecutive n (coalesced)
      uint32_t w4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w4[e] = (uint32_t)Wg[(8 * c16 + 2 * e) * N + n] | ((uint32_t)Wg[(8 * c16 + 2 * e + 1) * N + n] << 16);
      const int slab = c16 >> 3, c = c16 & 7;
      *reinterpret_cast<uint4*>(Bs + slab * BSLAB + n * 128 + ((c ^ (n & 7)) << 4)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor-core reads
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {                                       // TMA producer
      for (int i = UM_STAGES; i < my_tiles; ++i) {
        mbar_wait(&empty[i % UM_STAGES], ((uint32_t)(i / UM_STAGES) & 1u) ^ 1u);   // stage freed by tile i - STAGES
        produce(i);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {                                       // MMA issuer
      for (int i = 0; i < my_tiles; ++i) {
        const int s = i % UM_STAGES, a = i & 1;
        const uint32_t ph = (uint32_t)(i / UM_STAGES) & 1u, aph = (uint32_t)(i >> 1) & 1u;
        if (i >= 2) mbar_wait(&tempty[a], aph ^ 1u);       // epilogue drained accumulator a
        mbar_wait(&full[s], ph);                           // K tile landed
        tc_fence_after();
        const uint32_t a_base = smem_u32(As + s * SB), b_base = smem_u32(Bs);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {                   // K = 128 = 8 x 16; 32-byte steps inside a swizzle atom
          const uint32_t ao = (uint32_t)((kk >> 2) * UM_SLAB + (kk & 3) * 32);
          const uint32_t bo = (uint32_t)((kk >> 2) * BSLAB + (kk & 3) * 32);
          umma_bf16(tbase + (uint32_t)(a * N), desc_k_sw128(a_base + ao), desc_k_sw128(b_base + bo), IDESC,
                    kk > 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);                            // the stage is free once these MMAs are done
        umma_commit(&tfull[a]);                            // accumulator a is complete
      }
    }
  } else if (FUSED && warp == EPI_W1) {
    if (lane == 0) {                                       // store warp: the landed K and V tiles -> the caches
      for (int i = 0; i < my_tiles; ++i) {
        const int s = i % UM_STAGES;
        mbar_wait(&full[s], (uint32_t)(i / UM_STAGES) & 1u);
        const int tdst = (int)(p.t0 + (int64_t)(tile0 + i) * UM_TOK);   // rows >= t0 + n are out of the maps' bounds
        tma_store_3d(&fm.Kd, 0, tdst, u, As + s * SB);
        tma_store_3d(&fm.Kd, 64, tdst, u, As + s * SB + UM_SLAB);
        tma_store_3d(&fm.Vd, 0, tdst, u, As + s * SB + 2 * UM_SLAB);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the stage has been read
        mbar_arrive(&empty[s]);
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");           // writes complete before the trigger
    }
  } else {
    // epilogue: warp w >= 2 reads TMEM lane quadrant w % 4 (the lanes a warp
    // may access), columns [h * N/ES, (h+1) * N/ES) with h = (w - 2) / 4; all
    // of its loads are issued before one wait
    const int q = warp & 3, h = (warp - 2) >> 2;
    uint32_t* cb = p.codes + (int64_t)b * p.c_sb + (int64_t)g * p.c_sh;
    for (int i = 0; i < my_tiles; ++i) {
      const int a = i & 1;
      const uint32_t aph = (uint32_t)(i >> 1) & 1u;
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      uint32_t v[WE][32];
#pragma unroll
      for (int c = 0; c < WE; ++c)
        tmem_ld32_nowait(tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * N + (h * WE + c) * 32), v[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);              // accumulator a may be overwritten
      uint32_t words[WE];
#pragma unroll
      for (int c = 0; c < WE; ++c) {
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) w |= (uint32_t)(__uint_as_float(v[c][j]) >= 0.f) << j;   // Sign, BitPack
        words[c] = w;
      }
      const int64_t t = p.t0 + (int64_t)(tile0 + i) * UM_TOK + q * 32 + lane;
      if (t < p.t0 + p.n) {
        uint32_t* dst = cb + t * W + h * WE;
        if constexpr (WE % 4 == 0) {
          if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int c = 0; c < WE; c += 4)
              *reinterpret_cast<uint4*>(dst + c) = make_uint4(words[c], words[c + 1], words[c + 2], words[c + 3]);
          } else {
#pragma unroll
            for (int c = 0; c < WE; ++c) dst[c] = words[c];
          }
        } else if constexpr (WE == 2) {
          if ((reinterpret_cast<uintptr_t>(dst) & 7) == 0) *reinterpret_cast<uint2*>(dst) = make_uint2(words[0], words[1]);
          else { dst[0] = words[0]; dst[1] = words[1]; }
        } else {
#pragma unroll
          for (int c = 0; c < WE; ++c) dst[c] = words[c];
        }
      }
    }
  }
  // every role done: release TMEM, make the codes visible, trigger dependents
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(tmem_cols<N>()));
  }
  __threadfence();
  __syncthreads();
  griddep_launch_dependents();
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

template <int N, bool FUSED>
cudaError_t launch_n(const HashKeysParams& p, const CUtensorMap& map, const FusedMaps& fm, int64_t row_sb,
                     int64_t row_sh, cudaStream_t s) {
  const size_t smem = umma_smem_bytes<N, FUSED>();
  cudaError_t e = cudaFuncSetAttribute(hash_keys_umma_kernel<N, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int units = p.B * p.Hkv;
  const int ntiles = (int)((p.n + UM_TOK - 1) / UM_TOK);
  int per_unit = device_sm_count() / (units > 0 ? units : 1);   // one CTA per SM: fill the chip once
  if (per_unit < 1) per_unit = 1;
  if (per_unit > ntiles) per_unit = ntiles;
  const int tiles_per_cta = (ntiles + per_unit - 1) / per_unit;
  const int nx = (ntiles + tiles_per_cta - 1) / tiles_per_cta;
  hash_keys_umma_kernel<N, FUSED><<<dim3(nx, units), um_threads<N, FUSED>(), smem, s>>>(map, fm, p, row_sb, row_sh,
                                                                                         ntiles, tiles_per_cta);
  return cudaGetLastError();
}

template <bool FUSED>
cudaError_t dispatch_n(const HashKeysParams& p, const CUtensorMap& map, const FusedMaps& fm, int64_t row_sb,
                       int64_t row_sh, cudaStream_t s) {
  switch (p.rbits) {
    case 32: return launch_n<32, FUSED>(p, map, fm, row_sb, row_sh, s);
    case 64: return launch_n<64, FUSED>(p, map, fm, row_sb, row_sh, s);
    case 128: return launch_n<128, FUSED>(p, map, fm, row_sb, row_sh, s);
    case 256: return launch_n<256, FUSED>(p, map, fm, row_sb, row_sh, s);
  }
  return cudaErrorNotSupported;
}

// 3-D map {d, tokens, units} over a [B, H_kv, tokens, d] tensor whose batch
// stride is H_kv times its head stride (one unit stride)
bool map3d(EncodeTiledFn enc, CUtensorMap* m, const void* base, int64_t tokens, int units, int64_t st, int64_t sh,
           bool swz) {
  const cuuint64_t gdim[3] = {128, (cuuint64_t)tokens, (cuuint64_t)units};
  const cuuint64_t gstride[2] = {(cuuint64_t)(st * 2), (cuuint64_t)(sh * 2)};
  const cuuint32_t box[3] = {swz ? 64u : 128u, (cuuint32_t)UM_TOK, 1};
  const cuuint32_t estride[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gdim, gstride, box, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// bf16, d = 128, rbits in {32, 64, 128, 256}, and a K cache whose (b, g)
// strides are multiples of its row stride (one 2-D tensor map covers it);
// anything else -> cudaErrorNotSupported (the caller falls back).
cudaError_t launch_hash_keys_umma(const HashKeysParams& p, cudaStream_t s) {
  if (p.d != 128 || p.n <= 0) return p.n <= 0 ? cudaSuccess : cudaErrorNotSupported;
  if (p.rbits != 32 && p.rbits != 64 && p.rbits != 128 && p.rbits != 256) return cudaErrorNotSupported;
  const int64_t st = p.kv_st;
  if (st < 128 || (st * 2) % 16 || p.kv_sb % st || p.kv_sh % st || (reinterpret_cast<uintptr_t>(p.K) & 15))
    return cudaErrorNotSupported;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const int64_t row_sb = p.kv_sb / st, row_sh = p.kv_sh / st;
  const int64_t rows = (int64_t)(p.B - 1) * row_sb + (int64_t)(p.Hkv - 1) * row_sh + p.cap;
  if (rows <= 0 || rows >= ((int64_t)1 << 31)) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t gdim[2] = {128, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)(st * 2)};
  const cuuint32_t box[2] = {64, UM_TOK};
  const cuuint32_t estride[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p.K), gdim, gstride, box, estride,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  FusedMaps none;
  std::memset(&none, 0, sizeof(none));
  return dispatch_n<false>(p, map, none, row_sb, row_sh, s);
}

// NEXT-1 (hata_prefill_write): rows [0, n) of the chunk K_src / V_src ->
// rows [t0, t0 + n) of the K / V caches, and their codes, in one pass.
cudaError_t launch_prefill_write_umma(const HashKeysParams& p, const void* Ksrc, const void* Vsrc, int64_t ss_b,
                                      int64_t ss_h, int64_t ss_t, void* Vdst, cudaStream_t s) {
  if (p.d != 128 || p.n <= 0) return p.n <= 0 ? cudaSuccess : cudaErrorNotSupported;
  if (p.rbits != 32 && p.rbits != 64 && p.rbits != 128 && p.rbits != 256) return cudaErrorNotSupported;
  auto al = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; };
  if (!al(Ksrc) || !al(Vsrc) || !al(p.K) || !al(Vdst) || (ss_t * 2) % 16 || (p.kv_st * 2) % 16 || (ss_h * 2) % 16 ||
      (p.kv_sh * 2) % 16 || ss_b != (int64_t)p.Hkv * ss_h || p.kv_sb != (int64_t)p.Hkv * p.kv_sh || ss_t < 128 ||
      p.kv_st < 128)
    return cudaErrorNotSupported;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const int units = p.B * p.Hkv;
  CUtensorMap mk;
  FusedMaps fm;
  // destination maps end at row t0 + n of every unit: the tail tile's rows
  // past it are clipped by the TMA store (never written)
  if (!map3d(enc, &mk, Ksrc, p.n, units, ss_t, ss_h, true) || !map3d(enc, &fm.Vs, Vsrc, p.n, units, ss_t, ss_h, false) ||
      !map3d(enc, &fm.Kd, p.K, p.t0 + p.n, units, p.kv_st, p.kv_sh, true) ||
      !map3d(enc, &fm.Vd, Vdst, p.t0 + p.n, units, p.kv_st, p.kv_sh, false))
    return cudaErrorNotSupported;
  return dispatch_n<true>(p, mk, fm, 0, 0, s);
}

}  // namespace hata
