// Microbenchmark: issue rate of back-to-back tcgen05.mma (kind::f16, bf16 -> fp32) with no other
// work on the SM, for the shapes the attention kernel uses (SS M128 N128: S = Q K^T; TS M128 N128:
// O += P V) against the larger ones (SS M128 N256; cta_group::2 M256 N128 SS/TS).  Reports
// dense FLOP per clock per SM, to compare with the 8192 FLOP/clk/SM bf16 peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2502_12085_b200/csrc/sm100.cuh"

using namespace apb::sm100;

constexpr int kIters = 2048;  // groups of D/16 = 8 MMAs (K = 128 per group)

__device__ __forceinline__ void mma_ss2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma_ts2(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile("{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
               "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void cluster_arrive_wait() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// CG: cta_group; TS: A from TMEM; N: MMA N (per instruction, whole pair for CG = 2)
template <int CG, bool TS, int N, int COMMIT_EVERY = 0>
__global__ void __launch_bounds__(128, 1) umma_kernel(unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  constexpr int M = 128 * CG;
  constexpr int NB = N / CG;               // B rows held by this CTA
  constexpr int kSubA = 128 * 128;         // [128 rows][64 cols] bf16
  constexpr int kSubB = NB * 128;
  const uint32_t sA = smem_u32(smem), sB = sA + 2 * kSubA, bar = sB + 2 * kSubB;
  __shared__ uint32_t tmem_slot;
  for (int i = threadIdx.x; i < (2 * kSubA + 2 * kSubB) / 4; i += 128)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);  // small bf16 values
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 8, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_arrive_wait();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  constexpr uint32_t idesc_ss = idesc_bf16_f32(M, N, false, false);
  constexpr uint32_t idesc_ts = idesc_bf16_f32(M, N, false, true);
  if (threadIdx.x == 0 && rank == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
      const uint32_t dcol = (it & 1) * 256;  // two accumulators (N <= 256 columns each)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k / 4) * kSubA + (k % 4) * 32;
        const uint32_t offb = (k / 4) * kSubB + (k % 4) * 32;
        if (TS) {
          // A from TMEM columns [k*8, k*8+8) of the other accumulator slot; B MN-major-ish descriptor
          const uint64_t b = sdesc_sw128(sB + k * 2048 % kSubB, kSubB, 1024);
          if (CG == 1) mma_ts(tmem + dcol, tmem + (256 - dcol) + k * 8, b, idesc_ts, k > 0);
          else mma_ts2(tmem + dcol, tmem + (256 - dcol) + k * 8, b, idesc_ts, k > 0);
        } else {
          const uint64_t a = sdesc_sw128(sA + off, 16, 1024), b = sdesc_sw128(sB + offb, 16, 1024);
          if (CG == 1) mma_ss(tmem + dcol, a, b, idesc_ss, k > 0);
          else mma_ss2(tmem + dcol, a, b, idesc_ss, k > 0);
        }
        if (COMMIT_EVERY && (k + 1) % COMMIT_EVERY == 0) {  // commit to a never-awaited barrier
          if (CG == 1) mma_commit(bar + 8);
          else commit2(bar + 8);
        }
      }
    }
    if (CG == 1) mma_commit(bar);
    else commit2(bar);
    mbar_wait(bar, 0);
    const unsigned long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  } else if (CG == 2 && threadIdx.x == 0) {
    mbar_wait(bar, 0);  // the leader's multicast commit arrives here too
    cycles[blockIdx.x] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_arrive_wait();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Attention-shaped dependency chain without the softmax work (cta_group::1, 384 threads): two
// query tiles t; per KV step the MMA warp issues PV_t (8 TS MMAs, A = P_t from S_t's TMEM columns)
// then S_t(i+1) (8 SS MMAs) + commit(bS_t); the tile's softmax warpgroup (4 warps) waits bS_t and
// immediately arrives on bP_t (count 128, or one elected lane per warp); the MMA warp waits bP_t.
// MODE bit 0: sleeping waits (try_wait with suspend hint) in the MMA warp; bit 1: P in two halves.
__device__ __forceinline__ void bulk_load_g(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
template <int MODE>
__global__ void __launch_bounds__(384, 1) chain_kernel(unsigned long long* cycles, int steps, const uint8_t* src) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  constexpr int kSub = 128 * 128;
  const uint32_t sQ = smem_u32(smem), sK = sQ + 4 * kSub, sV = sK + 2 * kSub, sX = sV + 2 * kSub;
  const uint32_t bar = sX + ((MODE & 4) ? 4 * kSub : 0);
  __shared__ volatile int done_flag;
  auto bS = [&](int t) { return bar + 8 * t; };
  auto bP = [&](int t, int h) { return bar + 16 + 16 * t + 8 * h; };
  __shared__ uint32_t tmem_slot;
  for (int i = threadIdx.x; i < 8 * kSub / 4; i += 384)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    for (int t = 0; t < 2; ++t) {
      mbar_init(bS(t), 1);
      mbar_init(bP(t, 0), 128);
      mbar_init(bP(t, 1), 128);
    }
    mbar_init(bar + 48, 1);  // producer copies
    done_flag = 0;
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x / 32 == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_slot, 0);
  const int warp = threadIdx.x / 32;
  constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false), idPV = idesc_bf16_f32(128, 128, false, true);
  if (warp == 9) {
    unsigned long long t0 = clock64();
    auto wait = [&](uint32_t b, uint32_t ph) { if (MODE & 1) mbar_wait_sleep(b, ph); else mbar_wait(b, ph); };
    auto issue_S = [&](int t) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k / 4) * kSub + (k % 4) * 32;
          mma_ss(tmem + t * 128, sdesc_sw128(sQ + t * 2 * kSub + off, 16, 1024), sdesc_sw128(sK + off, 16, 1024), idS, k > 0);
        }
        mma_commit(bS(t));
      }
      __syncwarp();
    };
    for (int t = 0; t < 2; ++t) issue_S(t);
    for (int i = 0; i < steps; ++i) {
      for (int t = 0; t < 2; ++t) {
        for (int h = 0; h < 2; ++h) {
          if ((MODE & 2) || h == 0) wait(bP(t, h), i & 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int k = h * 4; k < h * 4 + 4; ++k)
              mma_ts(tmem + 256 + t * 128, tmem + t * 128 + k * 8, sdesc_sw128(sV + k * 2048, kSub, 1024), idPV, 1);
          }
          __syncwarp();
        }
        if (i + 1 < steps) issue_S(t);
      }
    }
    if (elect_one()) mma_commit(bS(0));
    __syncwarp();
    mbar_wait(bS(0), steps & 1);  // phase `steps` of bS(0): the final commit
    if (elect_one()) cycles[blockIdx.x] = clock64() - t0;
    done_flag = 1;
  } else if (warp == 10 && (MODE & 4)) {
    // TMA-like smem write stream: 4 x 16 KB bulk copies (L2-resident source) per round, waited on;
    // MODE & 8: pause between rounds to about 32 B/clk (the attention's K/V rate at full MMA speed)
    uint32_t ph = 0;
    while (!done_flag) {
      if (elect_one()) {
        mbar_arrive_expect_tx(bar + 48, 4 * kSub);
        for (int c = 0; c < 4; ++c) bulk_load_g(sX + c * kSub, src + (size_t)(blockIdx.x % 8) * 4 * kSub + c * kSub, kSub, bar + 48);
      }
      __syncwarp();
      mbar_wait(bar + 48, ph);
      ph ^= 1;
      if (MODE & 8) __nanosleep(1000);
    }
  } else if (warp < 8) {
    const int t = warp / 4;
    for (int i = 0; i < steps; ++i) {
      mbar_wait(bS(t), i & 1);
      tc_fence_after();
      tc_fence_before();
      mbar_arrive(bP(t, 0));
      if (MODE & 2) mbar_arrive(bP(t, 1));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int MODE>
void run_chain(const char* name, int sms) {
  auto kern = chain_kernel<MODE>;
  const int smem = 8 * 128 * 128 + ((MODE & 4) ? 4 * 128 * 128 : 0) + 64 + 1024;
  static uint8_t* src = nullptr;
  if (!src) { cudaMalloc(&src, 8 * 4 * 128 * 128); cudaMemset(src, 0x3c, 8 * 4 * 128 * 128); }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  cudaMemset(cyc, 0, sizeof(unsigned long long) * sms);
  const int steps = 512;
  kern<<<sms, 384, smem>>>(cyc, steps, src);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double csum = 0;
  for (int i = 0; i < sms; ++i) csum += h[i];
  const double flop = 2.0 * 2 * 2.0 * 128 * 128 * 128 * steps;  // 2 tiles x (S + PV) per step
  printf("%-28s %7.0f FLOP/clk/SM (%.3f of 8192)\n", name, flop / (csum / sms), flop / (csum / sms) / 8192.0);
  cudaFree(cyc);
}

template <int CG, bool TS, int N, int COMMIT_EVERY = 0>
void run(const char* name, int sms) {
  auto kern = umma_kernel<CG, TS, N, COMMIT_EVERY>;
  const int smem = 2 * 128 * 128 + 2 * (N / CG) * 128 + 64 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, kern, cyc);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaEventSynchronize(e1);
    if (err != cudaSuccess || e2 != cudaSuccess) {
      printf("%-28s launch error: %s / %s\n", name, cudaGetErrorString(err), cudaGetErrorString(e2));
      return;
    }
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double cmax = 0, csum = 0;
  int n = 0;
  for (int i = 0; i < sms; ++i)
    if (h[i]) { cmax = h[i] > cmax ? h[i] : cmax; csum += h[i]; ++n; }
  const double flop_pair = 2.0 * (128.0 * CG) * N * 128 * kIters;  // per issuing CTA (pair for CG = 2)
  const double per_sm_clk = flop_pair / CG / (csum / n);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-28s %7.0f FLOP/clk/SM (%.3f of 8192)  kernel %.3f ms -> %.0f TF/s over %d SMs\n", name, per_sm_clk,
         per_sm_clk / 8192.0, ms, flop_pair * (sms / CG) / (ms * 1e-3) / 1e12, sms);
  cudaFree(cyc);
}

// P-in-shared-memory pipeline (candidate attention restructure): per tile t and step i the
// "softmax" warpgroup waits S_t(i), arrives Sfree_t (the MMA warp may overwrite S_t at once),
// writes P_t (32 KB bf16, SW128 K-major) into shared memory with st.shared.v4, fences the async
// proxy and arrives P_t; the MMA warp issues S_t(i+1) on Sfree_t and PV_t(i) (SS: A = P_t from
// smem) on P_t.  MODE & 4: a concurrent 32 KB-per-round bulk-copy stream (the K/V TMA traffic).
template <int MODE>
__global__ void __launch_bounds__(384, 1) pchain_kernel(unsigned long long* cycles, int steps, const uint8_t* src) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  constexpr int kSub = 128 * 128;
  const uint32_t sQ = smem_u32(smem), sK = sQ + 4 * kSub, sV = sK + 2 * kSub, sP = sV + 2 * kSub, sX = sP + 4 * kSub;
  const uint32_t bar = sX + ((MODE & 4) ? 2 * kSub : 0);
  auto bS = [&](int t) { return bar + 8 * t; };
  auto bSf = [&](int t) { return bar + 16 + 8 * t; };
  auto bP = [&](int t) { return bar + 32 + 8 * t; };
  auto bPV = [&](int t) { return bar + 48 + 8 * t; };
  const uint32_t bX = bar + 64;
  __shared__ uint32_t tmem_slot;
  __shared__ volatile int done_flag;
  for (int i = threadIdx.x; i < 12 * kSub / 4; i += 384)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    for (int t = 0; t < 2; ++t) {
      mbar_init(bS(t), 1);
      mbar_init(bSf(t), 128);
      mbar_init(bP(t), 128);
      mbar_init(bPV(t), 1);
    }
    mbar_init(bX, 1);
    done_flag = 0;
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x / 32 == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_slot, 0);
  const int warp = threadIdx.x / 32;
  constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false), idPV = idesc_bf16_f32(128, 128, false, true);
  if (warp == 9) {
    const unsigned long long t0 = clock64();
    auto issue_S = [&](int t) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k / 4) * kSub + (k % 4) * 32;
          mma_ss(tmem + t * 128, sdesc_sw128(sQ + t * 2 * kSub + off, 16, 1024), sdesc_sw128(sK + off, 16, 1024), idS, k > 0);
        }
        mma_commit(bS(t));
      }
      __syncwarp();
    };
    auto issue_PV = [&](int t) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k / 4) * kSub + (k % 4) * 32;
          mma_ss(tmem + 256 + t * 128, sdesc_sw128(sP + t * 2 * kSub + off, 16, 1024),
                 sdesc_sw128(sV + k * 2048, kSub, 1024), idPV, 1);
        }
        mma_commit(bPV(t));
      }
      __syncwarp();
    };
    for (int t = 0; t < 2; ++t) issue_S(t);
    for (int i = 0; i < steps; ++i) {
      for (int t = 0; t < 2; ++t) {
        mbar_wait(bSf(t), i & 1);
        tc_fence_after();
        if (i + 1 < steps) issue_S(t);
      }
      for (int t = 0; t < 2; ++t) {
        mbar_wait(bP(t), i & 1);
        tc_fence_after();
        issue_PV(t);
      }
    }
    mbar_wait(bPV(1), (steps - 1) & 1);
    if (elect_one()) cycles[blockIdx.x] = clock64() - t0;
    done_flag = 1;
  } else if (warp == 10 && (MODE & 4)) {
    uint32_t ph = 0;
    while (!done_flag) {
      if (elect_one()) {
        mbar_arrive_expect_tx(bX, 2 * kSub);
        for (int c = 0; c < 2; ++c) bulk_load_g(sX + c * kSub, src + (size_t)(blockIdx.x % 8) * 2 * kSub + c * kSub, kSub, bX);
      }
      __syncwarp();
      mbar_wait(bX, ph);
      ph ^= 1;
    }
  } else if (warp < 8) {
    const int t = warp / 4, row = threadIdx.x % 128;
    for (int i = 0; i < steps; ++i) {
      mbar_wait(bS(t), i & 1);
      tc_fence_after();
      tc_fence_before();
      mbar_arrive(bSf(t));
      if (i > 0) mbar_wait(bPV(t), (i - 1) & 1);  // P_t(i-1) consumed
      // write this row's 128 bf16 P values (SW128 K-major: two [128][64] sub-tiles)
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int sub = j / 8, chunk = j % 8;
        const uint32_t a = sP + t * 2 * kSub + sub * kSub + row * 128 + ((chunk ^ (row & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(i + j), "r"(row), "r"(j), "r"(i) : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(bP(t));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int MODE>
void run_pchain(const char* name, int sms) {
  auto kern = pchain_kernel<MODE>;
  const int smem = 12 * 128 * 128 + ((MODE & 4) ? 2 * 128 * 128 : 0) + 128 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  static uint8_t* src = nullptr;
  if (!src) { cudaMalloc(&src, 8 * 4 * 128 * 128); cudaMemset(src, 0x3c, 8 * 4 * 128 * 128); }
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  cudaMemset(cyc, 0, sizeof(unsigned long long) * sms);
  const int steps = 512;
  kern<<<sms, 384, smem>>>(cyc, steps, src);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double csum = 0;
  for (int i = 0; i < sms; ++i) csum += h[i];
  const double flop = 2.0 * 2 * 2.0 * 128 * 128 * 128 * steps;
  printf("%-28s %7.0f FLOP/clk/SM (%.3f of 8192)\n", name, flop / (csum / sms), flop / (csum / sms) / 8192.0);
  cudaFree(cyc);
}

// SS MMA with M = 64 (cta_group::1): rate per SM relative to the 8192 FLOP/clk peak
template <int N>
__global__ void __launch_bounds__(128, 1) umma_m64_kernel(unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  constexpr int kSubA = 64 * 128, kSubB = N * 128;
  const uint32_t sA = smem_u32(smem), sB = sA + 2 * kSubA, bar = sB + 2 * kSubB;
  __shared__ uint32_t tmem_slot;
  for (int i = threadIdx.x; i < (2 * kSubA + 2 * kSubB) / 4; i += 128)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  constexpr uint32_t idesc = idesc_bf16_f32(64, N, false, false);
  if (threadIdx.x == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
      const uint32_t dcol = (it & 1) * 256;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k / 4) * kSubA + (k % 4) * 32, offb = (k / 4) * kSubB + (k % 4) * 32;
        mma_ss(tmem + dcol, sdesc_sw128(sA + off, 16, 1024), sdesc_sw128(sB + offb, 16, 1024), idesc, k > 0);
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int N>
void run_m64(const char* name, int sms) {
  auto kern = umma_m64_kernel<N>;
  const int smem = 2 * 64 * 128 + 2 * N * 128 + 64 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  kern<<<sms, 128, smem>>>(cyc);
  kern<<<sms, 128, smem>>>(cyc);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: error\n", name); return; }
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  const double flop = 2.0 * 64 * N * 128 * kIters;
  printf("%-28s %7.0f FLOP/clk/SM (%.3f of 8192)\n", name, flop / c, flop / c / 8192.0);
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sms &= ~1;
  run<1, false, 64>("cg1 SS M128 N64", sms);
  run<1, false, 128>("cg1 SS M128 N128", sms);
  run<1, false, 256>("cg1 SS M128 N256", sms);
  run<1, true, 128>("cg1 TS M128 N128", sms);
  run<2, false, 128>("cg2 SS M256 N128", sms);
  run<2, false, 256>("cg2 SS M256 N256", sms);
  run<2, true, 128>("cg2 TS M256 N128", sms);
  run<1, false, 128, 8>("cg1 SS N128 commit/8", sms);
  run<1, false, 128, 4>("cg1 SS N128 commit/4", sms);
  run<1, false, 128, 2>("cg1 SS N128 commit/2", sms);
  run<1, true, 128, 4>("cg1 TS N128 commit/4", sms);
  run<2, false, 128, 4>("cg2 SS N128 commit/4", sms);
  run_chain<0>("chain spin, P whole", sms);
  run_chain<1>("chain sleep, P whole", sms);
  run_chain<2>("chain spin, P halves", sms);
  run_chain<3>("chain sleep, P halves", sms);
  run_chain<6>("chain + smem writes (max)", sms);
  run_chain<14>("chain + smem writes (paced)", sms);
  run_pchain<0>("P-in-smem chain", sms);
  run_pchain<4>("P-in-smem chain + TMA stream", sms);
  run_m64<128>("cg1 SS M64 N128", sms);
  run_m64<256>("cg1 SS M64 N256", sms);
  return 0;
}
