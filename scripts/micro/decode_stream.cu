// Microbenchmark: the decode kernel's memory stream without its math.  A KV cache of
// `rows` x hk=8 x d=128 bf16 (K and V, [rows][hk][d] like the library's cache) is streamed by
// (split, KV head) CTAs in 64-key chunks, each CTA touching one 256-byte head slice of every
// 2 KB row — exactly decode_mma_kernel's access pattern — through
//   lsu : 16-byte cp.async per thread into a ring (what the kernel does),
//   tma : 2-D TMA boxes of 64 rows x 64 dims (128 B, SWIZZLE_128B), 2 per K/V chunk, one
//         issuing thread, full/empty mbarrier ring,
//   row : 2-D TMA boxes over whole 2 KB rows (8 rows x 64 dims, 16 boxes per K/V chunk) — the
//         contiguous-read ceiling of the same bytes,
// and reports TB/s of cache bytes read per launch (CUDA events, L2 flushed between launches).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o decode_stream decode_stream.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_2502_12085_b200/csrc/sm100.cuh"

using namespace apb::sm100;

constexpr int HK = 8, D = 128, CH = 64, NT = 256;

__device__ __forceinline__ void cp_async16(uint32_t d, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g) : "memory");
}

template <int S>
__global__ void __launch_bounds__(NT) lsu_kernel(const __nv_bfloat16* k, const __nv_bfloat16* v, int64_t rows,
                                                 int cps, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, j = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * cps;
  const int64_t nch_all = rows / CH;
  const int nch = (int)(c0 + cps <= nch_all ? cps : (nch_all > c0 ? nch_all - c0 : 0));
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  auto load = [&](int c, int s) {
    const int64_t r0 = (c0 + c) * CH;
    for (int i = tid; i < CH * 16; i += NT) {
      const int r = i / 16, cv = i % 16;
      const uint32_t off = r * 256 + ((cv ^ (r & 7)) << 4);
      cp_async16(sb + s * 32768 + off, k + (r0 + r) * (HK * D) + j * D + cv * 8);
      cp_async16(sb + s * 32768 + 16384 + off, v + (r0 + r) * (HK * D) + j * D + cv * 8);
    }
  };
  for (int s = 0; s < S - 1; ++s) {
    if (s < nch) load(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float acc = 0.f;
  for (int c = 0; c < nch; ++c) {
    if (c + S - 1 < nch) load(c + S - 1, (c + S - 1) % S);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    __syncthreads();
    acc += reinterpret_cast<const float*>(smem + (c % S) * 32768)[tid];
    __syncthreads();
  }
  if (acc == 12345.f) sink[0] = acc;
}

// TMA ring: stage = K chunk (2 boxes of 64 rows x 64 dims, 8 KB each) + V chunk (same)
template <int S, bool ROW>
__global__ void __launch_bounds__(NT) tma_kernel(const __grid_constant__ CUtensorMap tk,
                                                 const __grid_constant__ CUtensorMap tv, int64_t rows, int cps,
                                                 float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[S];
  const int tid = threadIdx.x, j = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * cps;
  const int64_t nch_all = rows / CH;
  const int nch = (int)(c0 + cps <= nch_all ? cps : (nch_all > c0 ? nch_all - c0 : 0));
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(static_cast<uint32_t>(__cvta_generic_to_shared(&full[s])), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int c, int s) {
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&full[s]));
    mbar_arrive_expect_tx(bar, 32768);
    const uint32_t dst = sb + s * 32768;
    if (!ROW) {
      const int r0 = (int)((c0 + c) * CH);
      tma_load_2d(dst, &tk, bar, j * D, r0);
      tma_load_2d(dst + 8192, &tk, bar, j * D + 64, r0);
      tma_load_2d(dst + 16384, &tv, bar, j * D, r0);
      tma_load_2d(dst + 24576, &tv, bar, j * D + 64, r0);
    } else {
      // same byte count from whole rows: 8 rows x 1024 dims = 16 boxes of 8 rows x 64 dims per K/V
      const int r0 = (int)(j * (rows / HK) + (c0 + c) * (CH / HK));
      for (int b = 0; b < 16; ++b) {
        tma_load_2d(dst + b * 1024, &tk, bar, b * 64, r0);
        tma_load_2d(dst + 16384 + b * 1024, &tv, bar, b * 64, r0);
      }
    }
  };
  if (tid == 0)
    for (int s = 0; s < S && s < nch; ++s) issue(s, s);
  float acc = 0.f;
  for (int c = 0; c < nch; ++c) {
    const int s = c % S;
    mbar_wait(static_cast<uint32_t>(__cvta_generic_to_shared(&full[s])), (c / S) & 1);
    acc += reinterpret_cast<const float*>(smem + s * 32768)[tid];
    __syncthreads();
    if (tid == 0 && c + S < nch) issue(c + S, s);
  }
  if (acc == 12345.f) sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap make_map(void* base, int64_t rows, int box_rows, bool swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)(HK * D), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(HK * D * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  return m;
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 131072;  // 8 hosts x 16K rows (L8 step)
  const size_t bytes = rows * HK * D * 2;
  __nv_bfloat16 *k, *v;
  float* sink;
  uint8_t* flush;
  cudaMalloc(&k, bytes);
  cudaMalloc(&v, bytes);
  cudaMalloc(&sink, 16);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(k, 0, bytes);
  cudaMemset(v, 0, bytes);
  const CUtensorMap tk = make_map(k, rows, 64, true), tv = make_map(v, rows, 64, true);
  const CUtensorMap rk = make_map(k, rows, 8, false), rv = make_map(v, rows, 8, false);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto launch) {
    float best = 1e9f, sum = 0.f;
    for (int it = 0; it < 12; ++it) {
      cudaMemsetAsync(flush, it, 256 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { best = ms < best ? ms : best; sum += ms; }
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); exit(1); }
    return std::make_pair(best, sum / 10);
  };
  const int64_t nch = rows / CH;
  printf("cache %.0f MiB (K+V), rows %lld, 2 KB rows, one 256 B head slice per CTA\n", 2.0 * bytes / 1048576,
         (long long)rows);
  for (int per_sm : {2, 3, 4, 6, 8}) {
    const int splits = (per_sm * 148 + HK - 1) / HK;
    const int cps = (int)((nch + splits - 1) / splits);
    const dim3 grid((unsigned)((nch + cps - 1) / cps), HK);
    auto rep = [&](const char* name, std::pair<float, float> t) {
      printf("%-10s ctas/sm-target %d grid %ux%u cps %d: best %.4f ms (%.2f TB/s)  mean %.4f ms (%.2f TB/s)\n", name,
             per_sm, grid.x, grid.y, cps, t.first, 2.0 * bytes / t.first / 1e9, t.second, 2.0 * bytes / t.second / 1e9);
    };
    cudaFuncSetAttribute(lsu_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768);
    cudaFuncSetAttribute(lsu_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768);
    rep("lsu S=2", time([&] { lsu_kernel<2><<<grid, NT, 2 * 32768>>>(k, v, rows, cps, sink); }));
    rep("lsu S=3", time([&] { lsu_kernel<3><<<grid, NT, 3 * 32768>>>(k, v, rows, cps, sink); }));
    cudaFuncSetAttribute(tma_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768 + 1024);
    cudaFuncSetAttribute(tma_kernel<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768 + 1024);
    cudaFuncSetAttribute(tma_kernel<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 1024);
    cudaFuncSetAttribute(tma_kernel<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768 + 1024);
    rep("tma S=2", time([&] { tma_kernel<2, false><<<grid, NT, 2 * 32768 + 1024>>>(tk, tv, rows, cps, sink); }));
    rep("tma S=3", time([&] { tma_kernel<3, false><<<grid, NT, 3 * 32768 + 1024>>>(tk, tv, rows, cps, sink); }));
    rep("tma S=4", time([&] { tma_kernel<4, false><<<grid, NT, 4 * 32768 + 1024>>>(tk, tv, rows, cps, sink); }));
    rep("row S=3", time([&] { tma_kernel<3, true><<<grid, NT, 3 * 32768 + 1024>>>(rk, rv, rows, cps, sink); }));
  }
  return 0;
}
