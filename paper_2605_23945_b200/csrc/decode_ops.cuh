// Parameter structs and launch helpers shared by the decode kernels and the C-ABI layer.
#pragma once
#include <stdint.h>

#include <utility>

#include "common.cuh"

namespace tps {

constexpr int kMaxPeers = 8;

// n fp32 buffers at base + i*stride (elements), summed in index order: the
// split-K partials of one projection, or one receive slot per TP rank. Fixed
// order keeps every rank of a TP group bitwise identical.
struct Src {
  const float* base;
  int n;
  long long stride;
};

// Cross-GPU completion counter wait: spin until *ctr >= (*epoch) * mult + add
// (or >= add when epoch is null). Counters only grow, so CUDA-graph replays
// need no host-side reset.
struct WaitSpec {
  const uint64_t* ctr;
  const uint64_t* epoch;
  uint64_t mult;
  uint64_t add;
};

// The last CTA of the launch (detected with the per-launch-site `done` counter,
// which it resets) issues the signals, so each rank contributes exactly one
// arrival per phase regardless of grid size / batch bucket.
struct SignalSpec {
  uint64_t* ctr[kMaxPeers];
  int n;
  unsigned int* done;
};

// Destination list for a reduce-and-push: the same [rows][cols] fp32 result is
// stored to every listed buffer (this rank's slot in each peer's receive area).
struct DstList {
  float* p[kMaxPeers];
  int n;
};

// Stochastic sampling (Gumbel-max with counter-based Philox4x32-10): a sample's sampler
// state is its key seeds[slot] and the position being sampled, so it migrates with the
// position (oracle/sampler_ref.py restates the arithmetic). seeds == NULL: greedy.
struct SamplerSpec {
  const uint64_t* seeds;
  const int* row_slot;
  const int* pos_by_slot;
  const int* row_pos;
  float inv_temp;
};

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ float gumbel_of(uint32_t x) {
  const float u = ((float)(x >> 8) + 0.5f) * (1.0f / 16777216.0f);
  return -logf(-logf(u));
}

struct ArgmaxCand {
  float val;
  int idx;
};

struct CandList {
  const ArgmaxCand* p[kMaxPeers];
  int n;
};

// The last CTA of the launch to get here (all threads of every CTA must call it)
// makes the launch's stores visible system-wide and adds 1 to every listed counter.
__device__ __forceinline__ void signal_last_cta(const SignalSpec& s) {
  if (s.n == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    // this CTA's (possibly remote) stores are ordered before its arrival at gpu scope; the
    // last CTA's system fence below is cumulative over everything it has observed, so one
    // fence.sc.sys per launch (not per CTA) publishes them to the peers
    __threadfence();
    const unsigned int nblocks = gridDim.x * gridDim.y * gridDim.z;
    const unsigned int prev = atomicAdd(s.done, 1u);
    if (prev == nblocks - 1) {
      *s.done = 0u;  // re-arm for the next launch / graph replay
      asm volatile("fence.acq_rel.sys;" ::: "memory");  // one system fence + relaxed adds = release per peer
      for (int i = 0; i < s.n; ++i) red_relaxed_sys_add(s.ctr[i], 1ull);
    }
  }
}

// ----------------------------------------------------- device step tracer (probe) ---
// When a trace buffer is registered (tps_trace_enable), thread 0 of block 0 of every traced
// launch writes [kind, t_entry, t_after_wait, t_exit] (%globaltimer ns) into the next free
// record; records land in launch order, so a graph replay reads back as an in-chain timeline
// (the latency each kernel adds inside a real step, PDL overlap included). Disabled: one
// load of a null pointer by one thread.
struct TraceBuf {
  uint64_t* p;
  unsigned int* ctr;
  unsigned int cap;
};
static __device__ TraceBuf g_trace_buf;  // one per translation unit, set by trace_register()
enum TraceKind : int {
  kTrEmbed = 1, kTrAddNorm, kTrReducePush, kTrQkvRope, kTrSilu, kTrArgmax1, kTrArgmax2, kTrEpoch,
  kTrGemm, kTrGemmSilu, kTrAttnSplit, kTrAttnCombine, kTrAttnBal, kTrAttnPrefill, kTrGemmPush, kTrGemv
};
__device__ __forceinline__ uint64_t trace_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned int trace_begin(int kind) {
  if (blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.x) return ~0u;
  const TraceBuf t = g_trace_buf;
  if (t.p == nullptr) return ~0u;
  const unsigned int slot = atomicAdd(t.ctr, 1u);
  if (slot >= t.cap) return ~0u;
  t.p[4 * slot] = (uint64_t)kind;
  t.p[4 * slot + 1] = trace_now();
  return slot;
}
__device__ __forceinline__ void trace_mark(unsigned int slot, int field) {
  if (slot != ~0u) g_trace_buf.p[4 * slot + field] = trace_now();
}
static inline int trace_register(uint64_t* p, unsigned int* ctr, unsigned int cap) {
  TraceBuf t{p, ctr, cap};
  return cudaMemcpyToSymbol(g_trace_buf, &t, sizeof(t)) == cudaSuccess ? 0 : -1;
}

// ----------------------------------------------- programmatic dependent launch
// Decode-step kernels are launched with the PDL attribute: each calls
// pdl_launch_dependents() early (the next kernel may start its prologue) and
// pdl_wait() before touching data produced or consumed by its predecessors.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();

template <typename... KArgs, typename... Args>
int launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return fail(kCuda, std::string("launch: ") + cudaGetErrorString(e));
  return kOk;
}

// launch_k with a thread-block cluster of cluster_x CTAs along x (DSMEM reductions).
template <typename... KArgs, typename... Args>
int launch_kcs(void (*kernel)(KArgs...), dim3 grid, dim3 block, int cluster_x, size_t smem, cudaStream_t st,
               bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return fail(kCuda, std::string("launch: ") + cudaGetErrorString(e));
  return kOk;
}

template <typename... KArgs, typename... Args>
int launch_kc(void (*kernel)(KArgs...), dim3 grid, dim3 block, int cluster_x, cudaStream_t st, bool pdl,
              Args... args) {
  return launch_kcs(kernel, grid, block, cluster_x, 0, st, pdl, args...);
}

}  // namespace tps
