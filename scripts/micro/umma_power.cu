// umma_power.cu — steady-state (power-capped) throughput of back-to-back tcgen05.mma streams:
// single-CTA M128 N128 (the attention's S = Q K^T shape, both operands from shared memory; and its
// TS form, O += P V with A from TMEM) against the CTA-pair forms (cta_group::2, M256 N128), which
// read half of B from each SM's shared memory.  Each configuration runs ~3 s on all SMs with
// random bf16 operands; NVML reports the median SM clock and board power of the second half.
// The question it answers: does halving the B-operand shared-memory reads per SM buy throughput
// under the 1000 W cap (energy per FLOP), i.e. is a 2-CTA attention worth building?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_power umma_power.cu -lnvidia-ml
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
#include <nvml.h>
#include "../../paper_2502_12085_b200/csrc/sm100.cuh"

using namespace apb::sm100;

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

template <int CG, bool TS>
__global__ void __launch_bounds__(128, 1) umma_kernel(int iters, uint32_t seed) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  constexpr int M = 128 * CG, N = 128;
  constexpr int NB = N / CG;
  constexpr int kSubA = 128 * 128, kSubB = NB * 128;
  const uint32_t sA = smem_u32(smem), sB = sA + 2 * kSubA, bar = sB + 2 * kSubB;
  __shared__ uint32_t tmem_slot;
  // random bf16 values in [-2, 2) (full mantissa toggling, as real activations)
  for (int i = threadIdx.x; i < (2 * kSubA + 2 * kSubB) / 4; i += 128) {
    uint32_t x = (i + blockIdx.x * 977u) * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    const uint32_t lo = 0x3f80u | (x & 0x407fu), hi = 0x3f80u | ((x >> 16) & 0x407fu);
    reinterpret_cast<uint32_t*>(smem)[i] = lo | (hi << 16);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    if (CG == 1) tmem_alloc<512>(smem_u32(&tmem_slot));
    else tmem_alloc_pair<512>(smem_u32(&tmem_slot));
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  uint32_t rank = 0;
  if (CG == 2) rank = cluster_ctarank();
  constexpr uint32_t idesc_ss = idesc_bf16_f32(M, N, false, false);
  constexpr uint32_t idesc_ts = idesc_bf16_f32(M, N, false, true);
  if (threadIdx.x == 0 && rank == 0) {
    for (int it = 0; it < iters; ++it) {
      const uint32_t dcol = (it & 1) * 256;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k / 4) * kSubA + (k % 4) * 32;
        const uint32_t offb = (k / 4) * kSubB + (k % 4) * 32;
        if (TS) {
          const uint64_t b = sdesc_sw128(sB + k * 2048 % kSubB, kSubB, 1024);
          if (CG == 1) mma_ts(tmem + dcol, tmem + (256 - dcol) + k * 8, b, idesc_ts, k > 0);
          else mma_ts2(tmem + dcol, tmem + (256 - dcol) + k * 8, b, idesc_ts, k > 0);
        } else {
          const uint64_t a = sdesc_sw128(sA + off, 16, 1024), b = sdesc_sw128(sB + offb, 16, 1024);
          if (CG == 1) mma_ss(tmem + dcol, a, b, idesc_ss, k > 0);
          else mma_ss2(tmem + dcol, a, b, idesc_ss, k > 0);
        }
      }
    }
    if (CG == 1) mma_commit(bar);
    else commit2(bar);
    mbar_wait(bar, 0);
  } else if (CG == 2 && threadIdx.x == 0) {
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if (CG == 1) tmem_dealloc<512>(tmem);
    else tmem_dealloc_pair<512>(tmem);
  }
}

template <int CG, bool TS>
void run(const char* name, int sms, nvmlDevice_t dev) {
  auto k = umma_kernel<CG, TS>;
  const int smem = (2 * 128 * 128 + 2 * (128 / CG) * 128) + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = CG;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  const int iters = 16384;  // per launch: 8 MMAs (K = 128) per iteration
  cudaLaunchKernelEx(&cfg, k, iters, 1u);  // warm
  cudaDeviceSynchronize();
  std::atomic<bool> stop{false};
  std::vector<unsigned> clk, pw;
  std::thread th([&] {
    while (!stop) {
      unsigned c = 0, p = 0;
      nvmlDeviceGetClockInfo(dev, NVML_CLOCK_SM, &c);
      nvmlDeviceGetPowerUsage(dev, &p);
      clk.push_back(c);
      pw.push_back(p);
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  });
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int launches = 0;
  auto t0 = std::chrono::steady_clock::now();
  cudaEventRecord(e0);
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 3.0) {
    for (int i = 0; i < 8; ++i, ++launches) cudaLaunchKernelEx(&cfg, k, iters, (unsigned)launches);
    cudaEventSynchronize(e0);  // keep the host close to the queue
    cudaDeviceSynchronize();
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  stop = true;
  th.join();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  // FLOP per launch: pairs x (2 M N K) per MMA group x iters, M = 128 CG
  const double flop = (double)(sms / CG) * 2.0 * (128.0 * CG) * 128.0 * 128.0 * iters * launches;
  const size_t h = clk.size() / 2;
  std::vector<unsigned> c2(clk.begin() + h, clk.end()), p2(pw.begin() + h, pw.end());
  std::sort(c2.begin(), c2.end());
  std::sort(p2.begin(), p2.end());
  printf("%-22s %8.1f TF/s  SM %u MHz  board %.0f W  (%d launches, %s)\n", name, flop / (ms * 1e-3) / 1e12,
         c2[c2.size() / 2], p2[p2.size() / 2] / 1e3, launches, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  nvmlInit();
  nvmlDevice_t dev;
  nvmlDeviceGetHandleByIndex(0, &dev);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sms &= ~1;
  for (int rep = 0; rep < 2; ++rep) {
    run<1, false>("cg1 SS M128 N128", sms, dev);
    run<2, false>("cg2 SS M256 N128", sms, dev);
    run<1, true>("cg1 TS M128 N128", sms, dev);
    run<2, true>("cg2 TS M256 N128", sms, dev);
  }
  nvmlShutdown();
  return 0;
}
