// Hardware probes for the HATA decode design on B200 (sm_100a). Not product code.
// Measures: shared-memory atomic histogram throughput, POPC/LOP3 issue rates for the
// Hamming score inner loop (naive XOR+POPC vs bit-plane mux + carry-save), cluster
// co-scheduling limits, L2 size, and streaming read bandwidth (LDG.128 vs cp.async.bulk).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// ---- 1. shared atomic histogram: values concentrated like D (mean 256, spread ~ +-40)
template <int MODE>
__global__ void k_hist(uint32_t* out, int iters, long long* cyc) {
  __shared__ uint32_t hist[8][520];
  for (int i = threadIdx.x; i < 8 * 520; i += blockDim.x) (&hist[0][0])[i] = 0;
  __syncthreads();
  uint32_t seed = hash32(blockIdx.x * 1024 + threadIdx.x);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t h = hash32(seed + it * 7919);
    // approx binomial-ish: sum of 4 bytes' popcounts around 16 -> spread
    uint32_t v = 200 + __popc(h) + __popc(h * 2654435761u) + ((h >> 3) & 63);
    if (MODE == 0) atomicAdd(&hist[0][v], 1u);
    else if (MODE == 1) atomicAdd(&hist[(threadIdx.x >> 5) & 7][v], 1u);
    else if (MODE == 2) { seed += v; }  // no atomic baseline
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  uint32_t s = seed;
  for (int i = threadIdx.x; i < 520; i += blockDim.x) s += hist[0][i] + hist[1][i];
  if (s == 0x12345678) out[0] = s;
}

// ---- 2. score inner loop on register-resident codes
template <int W>
__device__ __forceinline__ uint32_t score_naive(const uint32_t (&k)[W], const uint32_t (&q)[4][W]) {
  uint32_t d = 0;
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int w = 0; w < W; ++w) d += __popc(q[h][w] ^ k[w]);
  return d;
}
__device__ __forceinline__ uint32_t lop_mux(uint32_t k, uint32_t b, uint32_t a) {
  // k ? b : a  bitwise
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(k), "r"(b), "r"(a));
  return r;
}
__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(s) : "r"(a), "r"(b), "r"(c));
  asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(cy) : "r"(a), "r"(b), "r"(c));
}
// G=4, W=4: planes A_j (c bits), B_j ((G-c) bits), j<3
__device__ __forceinline__ uint32_t score_csa(const uint32_t (&k)[4], const uint32_t (&A)[3][4], const uint32_t (&B)[3][4]) {
  uint32_t m[3][4];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int w = 0; w < 4; ++w) m[j][w] = lop_mux(k[w], B[j][w], A[j][w]);
  // level 0: m0[0..3]
  uint32_t s0, c0, s0b, c0b;
  fa(m[0][0], m[0][1], m[0][2], s0, c0);
  s0b = s0 ^ m[0][3]; c0b = s0 & m[0][3];
  // level1 words: m1[0..3], c0, c0b
  uint32_t s1, c1, s1b, c1b;
  fa(m[1][0], m[1][1], m[1][2], s1, c1);
  fa(m[1][3], c0, c0b, s1b, c1b);
  uint32_t l1 = s1 ^ s1b, c1c = s1 & s1b;
  // level2 words: m2[0..3], c1, c1b, c1c
  uint32_t s2, c2, s2b, c2b, s2c, c2c;
  fa(m[2][0], m[2][1], m[2][2], s2, c2);
  fa(m[2][3], c1, c1b, s2b, c2b);
  fa(s2, s2b, c1c, s2c, c2c);
  // level3: c2, c2b, c2c
  uint32_t s3, c3;
  fa(c2, c2b, c2c, s3, c3);
  return __popc(s0b) + 2 * __popc(l1) + 4 * __popc(s2c) + 8 * __popc(s3) + 16 * __popc(c3);
}

template <int MODE>
__global__ void k_score(const uint4* __restrict__ codes, int n_per_thread, uint32_t* out, long long* cyc) {
  uint32_t q[4][4], A[3][4], B[3][4];
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int w = 0; w < 4; ++w) q[h][w] = hash32(h * 4 + w + 1);
#pragma unroll
  for (int w = 0; w < 4; ++w)
#pragma unroll
    for (int bit = 0; bit < 32; ++bit) {
      int c = 0;
      for (int h = 0; h < 4; ++h) c += (q[h][w] >> bit) & 1;
      int gc = 4 - c;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (bit == 0) { A[j][w] = 0; B[j][w] = 0; }
        A[j][w] |= ((c >> j) & 1u) << bit;
        B[j][w] |= ((gc >> j) & 1u) << bit;
      }
    }
  uint32_t acc = 0;
  uint32_t x = hash32(blockIdx.x * blockDim.x + threadIdx.x);
  long long t0 = clock64();
  for (int i = 0; i < n_per_thread; ++i) {
    uint32_t k[4];
    x = x * 1664525u + 1013904223u;
    k[0] = x; k[1] = x ^ 0x9e3779b9u; k[2] = x + 0x7f4a7c15u; k[3] = x * 3u;
    uint32_t d;
    if (MODE == 0) d = score_naive<4>(k, q);
    else if (MODE == 1) d = score_csa(k, A, B);
    else d = k[0] ^ k[1] ^ k[2] ^ k[3];
    acc += d;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x1234567) out[0] = acc;
}

// check csa == naive
__global__ void k_check(uint32_t* bad) {
  uint32_t q[4][4], A[3][4], B[3][4];
  for (int h = 0; h < 4; ++h) for (int w = 0; w < 4; ++w) q[h][w] = hash32(h * 4 + w + 11 + threadIdx.x);
  for (int w = 0; w < 4; ++w) for (int j = 0; j < 3; ++j) { A[j][w] = 0; B[j][w] = 0; }
  for (int w = 0; w < 4; ++w) for (int bit = 0; bit < 32; ++bit) {
    int c = 0; for (int h = 0; h < 4; ++h) c += (q[h][w] >> bit) & 1;
    for (int j = 0; j < 3; ++j) { A[j][w] |= ((c >> j) & 1u) << bit; B[j][w] |= (((4 - c) >> j) & 1u) << bit; }
  }
  for (int i = 0; i < 1000; ++i) {
    uint32_t k[4]; for (int w = 0; w < 4; ++w) k[w] = hash32(i * 4 + w + 12345 * threadIdx.x);
    if (score_naive<4>(k, q) != score_csa(k, A, B)) atomicAdd(bad, 1u);
  }
}

// ---- 3. streaming read bandwidth, LDG.128
__global__ void k_stream_ldg(const uint4* __restrict__ p, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldg(p + i), b = __ldg(p + i + stride), c = __ldg(p + i + 2 * stride), d = __ldg(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ b.z ^ b.w ^ c.x ^ c.w ^ d.y ^ d.z;
  }
  for (; i < n16; i += stride) { uint4 a = __ldg(p + i); acc ^= a.x ^ a.w; }
  if (acc == 0x12345) out[0] = acc;
}

// ---- 4. streaming via cp.async.bulk into a smem ring (1 producer thread)
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
template <int STAGES, int STAGE_BYTES>
__global__ void k_stream_bulk(const uint8_t* __restrict__ p, size_t bytes_per_cta, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[STAGES];
  const uint8_t* src = p + (size_t)blockIdx.x * bytes_per_cta;
  int nst = (int)(bytes_per_cta / STAGE_BYTES);
  if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0) for (int s = 0; s < STAGES && s < nst; ++s) { mbar_expect_tx(&bars[s], STAGE_BYTES); bulk_g2s(sm + s * STAGE_BYTES, src + (size_t)s * STAGE_BYTES, STAGE_BYTES, &bars[s]); }
  uint32_t acc = 0;
  for (int i = 0; i < nst; ++i) {
    int s = i % STAGES; uint32_t ph = (i / STAGES) & 1;
    mbar_wait(&bars[s], ph);
    const uint4* v = reinterpret_cast<const uint4*>(sm + s * STAGE_BYTES);
    for (int j = threadIdx.x; j < STAGE_BYTES / 16; j += blockDim.x) { uint4 a = v[j]; acc ^= a.x ^ a.w; }
    __syncthreads();
    if (threadIdx.x == 0 && i + STAGES < nst) { mbar_expect_tx(&bars[s], STAGE_BYTES); bulk_g2s(sm + s * STAGE_BYTES, src + (size_t)(i + STAGES) * STAGE_BYTES, STAGE_BYTES, &bars[s]); }
  }
  if (acc == 0x12345) out[0] = acc;
}

__global__ void __cluster_dims__(1, 1, 1) k_dummy_cluster() {}
__global__ void k_dummy() {}

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int l2 = 0, clk = 0, smem_optin = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  printf("{\"probe\":\"device\",\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"clock_khz\":%d,\"smem_optin\":%d}\n", pr.name, pr.multiProcessorCount, l2, clk, smem_optin);
  int nsm = pr.multiProcessorCount;
  uint32_t* dout; long long* dcyc; CK(cudaMalloc(&dout, 4096)); CK(cudaMalloc(&dcyc, 8 * 4096));
  std::vector<long long> hc(4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto med = [&](int n) { std::vector<long long> v(hc.begin(), hc.begin() + n); std::sort(v.begin(), v.end()); return (double)v[n / 2]; };

  // hist
  for (int threads : {256, 512}) {
    int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
      auto fn = mode == 0 ? k_hist<0> : (mode == 1 ? k_hist<1> : k_hist<2>);
      fn<<<nsm, threads>>>(dout, iters, dcyc); CK(cudaDeviceSynchronize());
      fn<<<nsm, threads>>>(dout, iters, dcyc); CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hc.data(), dcyc, 8 * nsm, cudaMemcpyDeviceToHost));
      double c = med(nsm);
      printf("{\"probe\":\"hist\",\"mode\":%d,\"threads\":%d,\"cyc_per_elem_per_sm\":%.4f}\n", mode, threads, c / ((double)iters * threads));
    }
  }
  // csa check
  CK(cudaMemset(dout, 0, 4)); k_check<<<1, 128>>>(dout); CK(cudaDeviceSynchronize());
  uint32_t bad; CK(cudaMemcpy(&bad, dout, 4, cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"csa_check\",\"mismatch\":%u}\n", bad);
  // score loops
  for (int threads : {256, 512, 1024}) {
    int n = 4096;
    for (int mode = 0; mode < 3; ++mode) {
      auto fn = mode == 0 ? k_score<0> : (mode == 1 ? k_score<1> : k_score<2>);
      fn<<<nsm, threads>>>(nullptr, n, dout, dcyc); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      fn<<<nsm, threads>>>(nullptr, n, dout, dcyc);
      cudaEventRecord(e1); CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(hc.data(), dcyc, 8 * nsm, cudaMemcpyDeviceToHost));
      double c = med(nsm);
      double tok = (double)n * threads * nsm;
      printf("{\"probe\":\"score\",\"mode\":\"%s\",\"threads\":%d,\"cyc_per_token_per_sm\":%.4f,\"gtok_s\":%.1f}\n",
             mode == 0 ? "naive" : (mode == 1 ? "csa" : "baseline"), threads, c / ((double)n * threads), tok / (ms * 1e-3) / 1e9);
    }
  }
  // clusters
  for (int cs : {2, 4, 8, 12, 16}) {
    for (int smem : {0, 100 * 1024, 200 * 1024}) {
      cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(cs * 16); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
      at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int ncl = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k_dummy, &cfg);
      printf("{\"probe\":\"cluster\",\"size\":%d,\"smem\":%d,\"max_active_clusters\":%d,\"err\":\"%s\"}\n", cs, smem, ncl, cudaGetErrorString(e));
      cudaGetLastError();
    }
  }
  // streaming
  size_t total = (size_t)1 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, total)); CK(cudaMemset(buf, 1, total));
  for (int grid : {nsm, 2 * nsm, 4 * nsm, 128}) {
    for (int threads : {256, 512}) {
      k_stream_ldg<<<grid, threads>>>((const uint4*)buf, total / 16, dout);
      CK(cudaDeviceSynchronize());
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); k_stream_ldg<<<grid, threads>>>((const uint4*)buf, total / 16, dout); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
      }
      printf("{\"probe\":\"stream_ldg\",\"grid\":%d,\"threads\":%d,\"GBps\":%.1f}\n", grid, threads, total / (best * 1e-3) / 1e9);
    }
  }
  for (int grid : {nsm, 128}) {
    constexpr int ST = 8, SB = 16384;
    size_t per = (total / grid) / SB * SB;
    cudaFuncSetAttribute(k_stream_bulk<ST, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB);
    k_stream_bulk<ST, SB><<<grid, 256, ST * SB>>>(buf, per, dout); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); k_stream_bulk<ST, SB><<<grid, 256, ST * SB>>>(buf, per, dout); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("{\"probe\":\"stream_bulk\",\"grid\":%d,\"stages\":%d,\"stage_bytes\":%d,\"GBps\":%.1f}\n", grid, ST, SB, per * grid / (best * 1e-3) / 1e9);
  }
  // small streams: 25 MB read (one CFG-4 layer) with 128 CTAs, rotating over 32 buffers -> latency/ramp effect
  {
    size_t sz = 16u << 20;  // 16 MB codes-equivalent
    constexpr int ST = 8, SB = 16384;
    size_t per = (sz / 128) / SB * SB;
    float best = 1e9;
    for (int r = 0; r < 32; ++r) {
      const uint8_t* src = buf + (size_t)(r % 32) * (sz) % (total - sz);
      cudaEventRecord(e0); k_stream_bulk<ST, SB><<<128, 256, ST * SB>>>(src, per, dout); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("{\"probe\":\"stream_bulk_16MB_128cta\",\"us\":%.2f,\"GBps\":%.1f}\n", best * 1e3, per * 128 / (best * 1e-3) / 1e9);
  }
  // launch overhead: empty kernel back to back
  {
    for (int i = 0; i < 10; ++i) k_dummy<<<148, 256>>>();
    cudaEventRecord(e0); for (int i = 0; i < 1000; ++i) k_dummy<<<148, 256>>>(); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"empty_launch_us\",\"us\":%.3f}\n", ms);
  }
  printf("{\"probe\":\"done\"}\n");
  return 0;
}
