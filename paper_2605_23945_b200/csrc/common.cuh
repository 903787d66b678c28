// Shared device/host helpers for libtpshift_b200 (sm_100a only).
//
// Every spin loop in this library is bounded by a watchdog (globaltimer based).
// A watchdog that fires does not trap (a trapped kernel leaves the device faulted,
// which on a shared GPU pool takes the GPU out of service): it prints, raises the
// library's abort word and abandons its wait; every other wait that has lasted
// over 1 ms polls the word and abandons too, so a protocol bug drains the queued
// work in seconds. The host sees the abort on its next checked call
// (tps_abort_status -> RuntimeError): a loud failure, results discarded.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#ifndef __CUDA_ARCH__
#define TPS_HOST_ONLY 1
#endif

namespace tps {

// ---------------------------------------------------------------- errors ---
enum Status : int {
  kOk = 0,
  kInvalid = -22,   // -EINVAL   -> tpshift ConfigError
  kPlan = -1001,    // -EPLAN    -> tpshift PlanVerificationError
  kCuda = -1002,    // CUDA runtime/driver failure; text via tps_last_error()
  kUnsupported = -95,
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define TPS_CHECK_ARG(cond, msg)                                   \
  do {                                                             \
    if (!(cond)) return ::tps::fail(::tps::kInvalid, (msg));       \
  } while (0)

#define TPS_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::tps::fail(::tps::kCuda, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

// Every decode-step kernel asks for the maximum shared-memory carveout, so consecutive
// kernels of a step never force an SM to drain and re-split L1/shared memory between
// launches (which would also serialise programmatic-dependent launches).
bool carveout_enabled();
#define TPS_MAX_CARVEOUT(kernel)                                                                   \
  do {                                                                                             \
    if (carveout_enabled())                                                                        \
      TPS_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,   \
                                        (int)cudaSharedmemCarveoutMaxShared));                     \
  } while (0)

#define TPS_LAUNCH_CHECK()                                                          \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess)                                                          \
      return ::tps::fail(::tps::kCuda, std::string("launch: ") + cudaGetErrorString(_e)); \
  } while (0)

constexpr int kNumSMs = 148;

// ------------------------------------------------------------- device util --
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Watchdog budget for every device-side wait: 20 s. Exceeding it raises the abort word.
constexpr uint64_t kWatchdogNs = 20ull * 1000ull * 1000ull * 1000ull;
// A wait polls the abort word once it has lasted this long (the fast path never reads it).
constexpr uint64_t kAbortPollNs = 1000ull * 1000ull;

// ------------------------------------------------------------ soft abort ---
// One host-mapped word (allocated by tps_init) shared by every translation unit: each TU
// holds its own copy of the pointer, set through the setter it registers here.
static __device__ unsigned int* g_abort_word = nullptr;
using AbortSetter = int (*)(unsigned int*);
int register_abort_setter(AbortSetter f);  // host side, abi.cu
namespace {
int set_abort_word_in_this_tu(unsigned int* p) {
  return (int)cudaMemcpyToSymbol(g_abort_word, &p, sizeof(p));
}
const int g_abort_registered = register_abort_setter(&set_abort_word_in_this_tu);
}  // namespace

__device__ __forceinline__ bool abort_raised() {
  const unsigned int* w = g_abort_word;
  return w != nullptr && *reinterpret_cast<const volatile unsigned int*>(w) != 0u;
}
static __device__ __noinline__ void raise_abort(unsigned int code) {
  unsigned int* w = g_abort_word;
  if (w != nullptr) {
    *reinterpret_cast<volatile unsigned int*>(w) = code;
    __threadfence_system();
  }
}
// true when a wait that started at t0 must be abandoned (watchdog fired here -- the caller
// prints first -- or raised elsewhere)
__device__ __forceinline__ bool wait_abandoned(uint64_t t0, bool* fired) {
  const uint64_t dt = globaltimer_ns() - t0;
  if (dt < kAbortPollNs) return false;
  if (abort_raised()) return true;
  if (dt > kWatchdogNs) {
    *fired = true;
    return true;
  }
  return false;
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// System-scope acquire load / release add for cross-GPU (NVLink P2P) flags.
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(uint64_t* p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Relaxed system-scope add. Preceded in program order by a fence.sc.sys
// (__threadfence_system) it forms a release pattern: signalling n peers costs one
// system fence instead of n (each red.release.sys is a fence of its own).
__device__ __forceinline__ void red_relaxed_sys_add(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Single-copy-atomic 8-byte system-scope stores / loads for the LL {value, tag} protocol.
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_relaxed_sys_v2u64(const uint64_t* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}

// Spin (one thread) until *p >= target; traps after the watchdog budget.
__device__ __forceinline__ void wait_counter_geq(const uint64_t* p, uint64_t target) {
  if (ld_acquire_sys(p) >= target) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys(p) < target) {
    __nanosleep(64);
    bool fired = false;
    if (wait_abandoned(t0, &fired)) {
      if (fired) {
        printf("tps watchdog: counter %p stuck at %llu < %llu\n", (const void*)p,
               (unsigned long long)ld_acquire_sys(p), (unsigned long long)target);
        raise_abort(1);
      }
      return;
    }
  }
}

// ----------------------------------------------------------- mbarrier/TMA --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait on an mbarrier phase (try_wait sleeps in hardware between polls).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try_wait(bar, parity)) {
    bool fired = false;
    if (wait_abandoned(t0, &fired)) {
      if (fired) {
        printf("tps watchdog: mbarrier wait timed out (block %d thread %d)\n", blockIdx.x, threadIdx.x);
        raise_abort(2);
      }
      return;
    }
  }
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 1-D bulk copies (TMA engine, no tensor map) between global and shared memory.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ----------------------------------------------------------------- tcgen05 --
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

}  // namespace tps
