// Dev microbenchmark: HBM streaming rate of a persistent 148-CTA grid whose producer warp
// TMA-loads weight boxes [box_rows x 64] (SWIZZLE_128B) into a ring that consumer warps
// release immediately. Measures the weight-stream pattern of csrc/persist.cu in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tsb tools/cuda/tma_stream_bench.cu -lcuda
//   /tmp/tsb <box_rows> <boxes_per_stage> <stages> <row_mode: 0 = unit-major (16-row units over K), 1 = k-major>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su32(d)), "l"((uint64_t)m), "r"(su32(b)), "r"(c0), "r"(c1) : "memory");
}

__device__ __forceinline__ void tma3d(void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(su32(d)), "l"((uint64_t)m), "r"(su32(b)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

__global__ void __launch_bounds__(288, 1) stream(const __grid_constant__ CUtensorMap tm, int rows, int K, int box_rows,
                                                 int bps, int stages, int mode, int reps, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int sbytes = box_rows * 128 * bps;
  uint64_t* full = (uint64_t*)(ring + stages * sbytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int units = rows / box_rows;           // row blocks
  const int kchunks = K / 64;                  // boxes per row block
  const long long total = (long long)units * kchunks / bps;  // stages
  const long long lo = (long long)blockIdx.x * total / gridDim.x, hi = (long long)(blockIdx.x + 1) * total / gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t it = 0;
  if (warp == 8) {
    if (lane) return;
    for (int r = 0; r < reps; ++r)
      for (long long s = lo; s < hi; ++s, ++it) {
        const uint32_t slot = it % stages;
        if (it >= (uint32_t)stages) wait(&empty[slot], ((it / stages) + 1) & 1);
        arrive_tx(&full[slot], sbytes);
        if (mode == 2) {  // one 3-D box: [nchunk = bps][box_rows][64], unit-major
          const int units = rows / box_rows, spu = kchunks / bps;
          const int u = (int)(s / spu), kc = (int)(s % spu) * bps;
          tma3d(ring + slot * sbytes, &tm, &full[slot], 0, u * box_rows, kc);
          continue;
        }
        for (int j = 0; j < bps; ++j) {
          const long long box = s * bps + j;
          int u, kc;
          if (mode == 0) { u = (int)(box / kchunks); kc = (int)(box % kchunks); }
          else { kc = (int)(box / units); u = (int)(box % units); }
          tma2d(ring + slot * sbytes + j * box_rows * 128, &tm, &full[slot], kc * 64, u * box_rows);
        }
      }
    return;
  }
  unsigned long long acc = 0;
  for (int r = 0; r < reps; ++r)
    for (long long s = lo; s < hi; ++s, ++it) {
      const uint32_t slot = it % stages;
      wait(&full[slot], (it / stages) & 1);
      acc += *(volatile uint32_t*)(ring + slot * sbytes + warp * 64 + lane * 4);
      __syncwarp();
      if (lane == 0) arrive(&empty[slot]);
    }
  if (acc == 0x12345) *sink = acc;
}

__global__ void fill(uint32_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 12345u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = x & 0x3fff3fffu;  // finite bf16 pairs, incompressible
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int box_rows = argc > 1 ? atoi(argv[1]) : 16, bps = argc > 2 ? atoi(argv[2]) : 4;
  const int stages = argc > 3 ? atoi(argv[3]) : 12, mode = argc > 4 ? atoi(argv[4]) : 0;
  const int rows = 37888, K = 4096;  // 310 MB (> L2); K / 64 divisible by every chunk count tested
  void* w;
  cudaMalloc(&w, (size_t)rows * K * 2);
  fill<<<1024, 256>>>((uint32_t*)w, (size_t)rows * K / 2);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
  CUresult rc;
  if (mode == 2) {  // dims {64, rows, K/64}, strides {2K, 128}: smem [chunk][row][64] (row-indexed swizzle)
    cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)K / 64}, s3[2] = {(cuuint64_t)K * 2, 128};
    cuuint32_t b3[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)bps}, e3[3] = {1, 1, 1};
    rc = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    rc = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (rc) { printf("encode failed %d\n", (int)rc); return 1; }
  const int smem = stages * box_rows * 128 * bps + 2048 + 1024;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int reps = 4;
  stream<<<148, 288, smem>>>(tm, rows, K, box_rows, bps, stages, mode, 1, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  stream<<<148, 288, smem>>>(tm, rows, K, box_rows, bps, stages, mode, reps, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)rows * K * 2 * reps;
  printf("box %3d rows x 64, %d boxes/stage (%5d B), %2d stages (%6d B ring), mode %d: %7.1f GB/s  err=%s\n", box_rows, bps,
         box_rows * 128 * bps, stages, stages * box_rows * 128 * bps, mode, bytes / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
