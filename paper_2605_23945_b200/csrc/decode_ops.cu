// Memory-bound decode-step kernels around the tcgen05 projections:
// embedding gather, residual add + RMSNorm (the consumer of O/down partials and
// of the TP allreduce), fused QKV bias + RoPE + paged-KV append, SiLU*up, the
// vocab-parallel greedy argmax with its cross-rank reduce, and the TP
// reduce-and-push (one-shot allreduce over NVLink P2P stores).
//
// At tail batch sizes these kernels are latency-bound, so they (1) sum split /
// rank partials from strided sources with all loads issued before the adds,
// (2) use programmatic dependent launch so their launch and prologue overlap
// the previous kernel, and (3) keep grids wide enough to spread across SMs.
//
// Batch rows are indirected through row_slot[b] -> sample slot; per-slot state
// (position, page table, token history) stays where it is when the batch is
// compacted after completions, so a CUDA-graph replay only needs a new
// row_slot vector. row_slot[b] < 0 marks a padding row of a graph bucket.
#include <stdlib.h>

#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "decode_ops.cuh"

namespace tps {

static bool g_pdl = true;
static bool g_carveout = [] {
  const char* e = getenv("TPS_CARVEOUT");
  return !(e && e[0] == '0');
}();
bool carveout_enabled() { return g_carveout; }
bool pdl_enabled() { return g_pdl; }
void set_pdl(bool on) { g_pdl = on; }

__device__ __forceinline__ void do_wait(const WaitSpec& w) {
  if (w.ctr == nullptr) return;
  if (threadIdx.x == 0) {
    const uint64_t target = w.add + (w.epoch ? (*(volatile const uint64_t*)w.epoch) * w.mult : 0ull);
    wait_counter_geq(w.ctr, target);
  }
  __syncthreads();
}

__device__ __forceinline__ void do_signal(const SignalSpec& s) { signal_last_cta(s); }

// sum_{i<n} base[i*stride + off] in index order, loads batched NB at a time (one L2
// round trip for up to NB split / rank partials)
template <int NB = 8>
__device__ __forceinline__ float4 src_sum4(const Src& s, long long off4) {
  const float4* b = reinterpret_cast<const float4*>(s.base) + off4;
  const long long st4 = s.stride / 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = 0; i0 < s.n; i0 += NB) {
    float4 v[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (i0 + j < s.n) v[j] = b[(long long)(i0 + j) * st4];
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (i0 + j < s.n) {
        acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w;
      }
  }
  return acc;
}

__device__ __forceinline__ float src_sum(const Src& s, long long off) {
  const float* b = s.base + off;
  float acc = 0.f;
  for (int i0 = 0; i0 < s.n; i0 += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (i0 + j < s.n) v[j] = b[(long long)(i0 + j) * s.stride];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (i0 + j < s.n) acc += v[j];
  }
  return acc;
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0.f;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  const float r = red[0];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------ embedding ---
// resid[b][:] = E[history[slot][pos]][:]  (replicated vocab table, bf16 -> fp32)
__global__ void embed_kernel(const int* __restrict__ row_slot, const int* __restrict__ pos_by_slot,
                             const int* __restrict__ row_pos, const int* __restrict__ history, int hist_ld,
                             const __nv_bfloat16* __restrict__ table, int H, float* __restrict__ resid) {
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrEmbed);
  pdl_wait();
  trace_mark(trs, 2);
  const int b = blockIdx.x;
  const int slot = row_slot[b];
  int tok = 0;
  if (slot >= 0) tok = history[(size_t)slot * hist_ld + (row_pos ? row_pos[b] : pos_by_slot[slot])];
  const __nv_bfloat162* src = reinterpret_cast<const __nv_bfloat162*>(table + (size_t)tok * H);
  float2* dst = reinterpret_cast<float2*>(resid + (size_t)b * H);
  for (int i = threadIdx.x; i < H / 2; i += blockDim.x) dst[i] = __bfloat1622float2(src[i]);
  trace_mark(trs, 3);
}

// ------------------------------------------------- residual add + RMSNorm ---
// resid[b] += sum_i src_i[b] (index order); out[b] = bf16(resid * rstd * w)
constexpr int kNormThreads = 512;
constexpr int kNormVec = 4;  // float4 per thread held in registers (H <= 8192)
template <int NB>
__global__ void __launch_bounds__(kNormThreads) add_norm_kernel(float* __restrict__ resid, Src src,
                                                                WaitSpec wait,
                                                                const __nv_bfloat16* __restrict__ w, float eps,
                                                                int H, __nv_bfloat16* __restrict__ out, int ldo) {
  __shared__ float red[32];
  const int b = blockIdx.x;
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrAddNorm);
  pdl_wait();
  do_wait(wait);
  trace_mark(trs, 2);
  float4* r4 = reinterpret_cast<float4*>(resid + (size_t)b * H);
  const int H4 = H / 4;
  float4 v[kNormVec];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kNormVec; ++j) {
    const int i = threadIdx.x + j * kNormThreads;
    if (i < H4) {
      float4 x = r4[i];
      if (src.n > 0) {
        const float4 p = src_sum4<NB>(src, (long long)b * H4 + i);
        x.x += p.x; x.y += p.y; x.z += p.z; x.w += p.w;
        r4[i] = x;
      }
      v[j] = x;
      ss += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
    }
  }
  ss = block_sum<kNormThreads>(ss, red);
  const float rstd = rsqrtf(ss / (float)H + eps);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + (size_t)b * ldo);
  const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(w);
#pragma unroll
  for (int j = 0; j < kNormVec; ++j) {
    const int i = threadIdx.x + j * kNormThreads;
    if (i < H4) {
      const float2 w01 = __bfloat1622float2(wp[2 * i]);
      const float2 w23 = __bfloat1622float2(wp[2 * i + 1]);
      o[2 * i] = __floats2bfloat162_rn(v[j].x * rstd * w01.x, v[j].y * rstd * w01.y);
      o[2 * i + 1] = __floats2bfloat162_rn(v[j].z * rstd * w23.x, v[j].w * rstd * w23.y);
    }
  }
  trace_mark(trs, 3);
}

// ------------------------------------- residual add + RMSNorm, LL sources ---
// Same as add_norm_kernel, but the n sources are the TP peers' fused-projection slots in
// LL form: uint64 {fp32 bits, tag} written by the producers' epilogues. Each thread polls
// its own elements until every tag equals (*epoch) * mult + add (watchdog-bounded), then
// sums the sources in index order: no counters, no fences on the critical path.
__device__ __forceinline__ bool ll_ok(const ulonglong2& a, const ulonglong2& c, uint32_t want) {
  return (uint32_t)(a.x >> 32) == want && (uint32_t)(a.y >> 32) == want && (uint32_t)(c.x >> 32) == want &&
         (uint32_t)(c.y >> 32) == want;
}

// Loads of NB sources are issued together (one L2 round trip per batch when the data is
// already there); a source whose tags are not yet current is re-polled on its own.
template <int NB = 8>
__device__ __forceinline__ float4 ll_sum4(const uint64_t* base, int n, long long stride, long long off4,
                                          uint32_t want) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = 0; i0 < n; i0 += NB) {
    ulonglong2 a[NB], c[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (i0 + j < n) {
        const uint64_t* p = base + (long long)(i0 + j) * stride + off4 * 4;
        a[j] = ld_relaxed_sys_v2u64(p);
        c[j] = ld_relaxed_sys_v2u64(p + 2);
      }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (i0 + j < n) {
        if (!ll_ok(a[j], c[j], want)) {
          const uint64_t* p = base + (long long)(i0 + j) * stride + off4 * 4;
          const uint64_t t0 = globaltimer_ns();
          do {
            bool fired = false;
            if (wait_abandoned(t0, &fired)) {
              if (fired) {
                printf("tps watchdog: LL source %d of %d (base %p, element %lld) tag %u != %u\n", i0 + j, n,
                       (const void*)base, off4 * 4, (unsigned)(a[j].x >> 32), want);
                raise_abort(3);
              }
              break;
            }
            a[j] = ld_relaxed_sys_v2u64(p);
            c[j] = ld_relaxed_sys_v2u64(p + 2);
          } while (!ll_ok(a[j], c[j], want));
        }
        acc.x += __uint_as_float((uint32_t)a[j].x);
        acc.y += __uint_as_float((uint32_t)a[j].y);
        acc.z += __uint_as_float((uint32_t)c[j].x);
        acc.w += __uint_as_float((uint32_t)c[j].y);
      }
  }
  return acc;
}

__global__ void __launch_bounds__(kNormThreads) add_norm_ll_kernel(float* __restrict__ resid,
                                                                   const uint64_t* __restrict__ ll, int nsrc,
                                                                   long long stride, const uint64_t* epoch,
                                                                   uint32_t mult, uint32_t add,
                                                                   const __nv_bfloat16* __restrict__ w, float eps,
                                                                   int H, __nv_bfloat16* __restrict__ out, int ldo,
                                                                   unsigned long long* ctr, unsigned long long bump) {
  __shared__ float red[32];
  const int b = blockIdx.x;
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrAddNorm);
  pdl_wait();
  trace_mark(trs, 2);
  const uint32_t want = (uint32_t)(*(volatile const uint64_t*)epoch * mult + add);
  // keep this phase's arrival counter at epoch * tp as if the counter protocol had run
  // (steps of one TP layout may use either protocol: B > 64 and chunked prefill push)
  if (ctr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(ctr, bump);
  float4* r4 = reinterpret_cast<float4*>(resid + (size_t)b * H);
  const int H4 = H / 4;
  float4 v[kNormVec];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kNormVec; ++j) {
    const int i = threadIdx.x + j * kNormThreads;
    if (i < H4) {
      float4 x = r4[i];
      const float4 p = ll_sum4(ll, nsrc, stride, (long long)b * H4 + i, want);
      x.x += p.x; x.y += p.y; x.z += p.z; x.w += p.w;
      r4[i] = x;
      v[j] = x;
      ss += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
    }
  }
  ss = block_sum<kNormThreads>(ss, red);
  const float rstd = rsqrtf(ss / (float)H + eps);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + (size_t)b * ldo);
  const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(w);
#pragma unroll
  for (int j = 0; j < kNormVec; ++j) {
    const int i = threadIdx.x + j * kNormThreads;
    if (i < H4) {
      const float2 w01 = __bfloat1622float2(wp[2 * i]);
      const float2 w23 = __bfloat1622float2(wp[2 * i + 1]);
      o[2 * i] = __floats2bfloat162_rn(v[j].x * rstd * w01.x, v[j].y * rstd * w01.y);
      o[2 * i + 1] = __floats2bfloat162_rn(v[j].z * rstd * w23.x, v[j].w * rstd * w23.y);
    }
  }
  trace_mark(trs, 3);
}

// ------------------------------- residual add + RMSNorm, cluster of 8 CTAs ---
// One row is split over a cluster of kNormCluster CTAs (each owns H / 8 columns), so the
// partial sums -- split-K partials, or the tp x splits slots of a fused TP allreduce,
// plain fp32 or LL {value, tag} -- are read by 8 SMs instead of one; the row's sum of
// squares is reduced through distributed shared memory in fixed rank order (identical on
// every CTA and every TP rank). LL: see add_norm_ll_kernel.
constexpr int kNormCluster = 8;
constexpr int kNormCThreads = 128;
constexpr int kNormCVec = 2;  // float4 per thread: H <= 8 * 128 * 2 * 4 = 8192
template <bool LL>
__global__ void __launch_bounds__(kNormCThreads)
    add_norm_cluster_kernel(float* __restrict__ resid, Src src, WaitSpec wait, const uint64_t* __restrict__ ll,
                            int nll, long long ll_stride, const uint64_t* epoch, uint32_t mult, uint32_t add,
                            unsigned long long* ctr, unsigned long long bump, const __nv_bfloat16* __restrict__ w,
                            float eps, int H, __nv_bfloat16* __restrict__ out, int ldo) {
  __shared__ float red[kNormCThreads / 32];
  __shared__ float s_part;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int b = blockIdx.y;
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrAddNorm);
  pdl_wait();
  if constexpr (!LL) do_wait(wait);
  trace_mark(trs, 2);
  uint32_t want = 0;
  if constexpr (LL) {
    want = (uint32_t)(*(volatile const uint64_t*)epoch * mult + add);
    if (ctr && crank == 0 && b == 0 && threadIdx.x == 0) atomicAdd(ctr, bump);
  }
  const int H4 = H / 4;
  const int per = (H4 + kNormCluster - 1) / kNormCluster;
  const int lo = crank * per, hi = min(H4, lo + per);
  float4* r4 = reinterpret_cast<float4*>(resid + (size_t)b * H);
  float4 v[kNormCVec];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kNormCVec; ++j) {
    const int i = lo + threadIdx.x + j * kNormCThreads;
    if (i < hi) {
      float4 x = r4[i];
      float4 p;
      if constexpr (LL) p = ll_sum4(ll, nll, ll_stride, (long long)b * H4 + i, want);
      else p = src.n > 0 ? src_sum4<16>(src, (long long)b * H4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (LL || src.n > 0) {
        x.x += p.x; x.y += p.y; x.z += p.z; x.w += p.w;
        r4[i] = x;
      }
      v[j] = x;
      ss += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kNormCThreads / 32; ++i) t += red[i];
    s_part = t;
  }
  cluster.sync();
  float tot = 0.f;
#pragma unroll
  for (int r = 0; r < kNormCluster; ++r) tot += *cluster.map_shared_rank(&s_part, r);
  const float rstd = rsqrtf(tot / (float)H + eps);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + (size_t)b * ldo);
  const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(w);
#pragma unroll
  for (int j = 0; j < kNormCVec; ++j) {
    const int i = lo + threadIdx.x + j * kNormCThreads;
    if (i < hi) {
      const float2 w01 = __bfloat1622float2(wp[2 * i]);
      const float2 w23 = __bfloat1622float2(wp[2 * i + 1]);
      o[2 * i] = __floats2bfloat162_rn(v[j].x * rstd * w01.x, v[j].y * rstd * w01.y);
      o[2 * i + 1] = __floats2bfloat162_rn(v[j].z * rstd * w23.x, v[j].w * rstd * w23.y);
    }
  }
  cluster.sync();  // peers may still be reading this CTA's partial
  trace_mark(trs, 3);
}

// ------------------------------------------- TP one-shot allreduce (push) ---
// Sum this rank's split-K partials and store the [rows][cols] result into this
// rank's slot of every TP peer's receive area (NVLink P2P stores), then signal.
constexpr int kPushBlocks = 64;
__global__ void __launch_bounds__(256) reduce_push_kernel(Src src, DstList dst, long long n4, SignalSpec sig) {
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrReducePush);
  pdl_wait();
  trace_mark(trs, 2);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = src_sum4(src, i);
    for (int d = 0; d < dst.n; ++d) reinterpret_cast<float4*>(dst.p[d])[i] = v;
  }
  do_signal(sig);
  trace_mark(trs, 3);
}

// LL form: sum the split partials, store {value, tag} pairs to every destination (no signal:
// the consumer polls the tags). Used for mid-size tail batches, where pushing every split
// partial from the projection epilogue would multiply the NVLink bytes by the split count.
__global__ void __launch_bounds__(256) reduce_push_ll_kernel(Src src, DstList dst, long long n4,
                                                             const uint64_t* epoch, uint32_t mult, uint32_t add) {
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrReducePush);
  pdl_wait();
  trace_mark(trs, 2);
  const uint64_t tag = (uint64_t)((uint32_t)(*(volatile const uint64_t*)epoch * mult + add)) << 32;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = src_sum4(src, i);
    for (int d = 0; d < dst.n; ++d) {
      uint64_t* o = reinterpret_cast<uint64_t*>(dst.p[d]) + 4 * i;
      st_relaxed_sys_u64(o, tag | __float_as_uint(v.x));
      st_relaxed_sys_u64(o + 1, tag | __float_as_uint(v.y));
      st_relaxed_sys_u64(o + 2, tag | __float_as_uint(v.z));
      st_relaxed_sys_u64(o + 3, tag | __float_as_uint(v.w));
    }
  }
  trace_mark(trs, 3);
}

// ---------------------------------------------- QKV bias + RoPE + KV append ---
// partial layout [split][B][Nqkv] with Nqkv = (nq + 2 nkv) * D, rows ordered
// [q heads | k heads | v heads] (canonical shard layout). RoPE is the
// rotate-half form used by Llama/Qwen2 with a host-built fp32 cos/sin table.
// KV cache per layer: [num_pages][nkv][P][D] bf16. One warp per (row, head).
// NV series of split partials summed together: all NV x 8 loads of a batch are in flight
// at once (one L2 round trip per 8 splits however many series a thread needs).
template <int NV>
__device__ __forceinline__ void src_sum_multi(const Src& s, const long long (&off)[NV], float (&out)[NV]) {
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = 0.f;
  for (int i0 = 0; i0 < s.n; i0 += 8) {
    float v[NV][8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (i0 + j < s.n) v[k][j] = s.base[(long long)(i0 + j) * s.stride + off[k]];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (i0 + j < s.n) out[k] += v[k][j];
  }
}

// One thread per (row, head, rotary pair i < D/2): every split partial of the pair is
// loaded in one batch, so a TP-sharded QKV with many splits costs one L2 round trip.
__global__ void __launch_bounds__(128) qkv_rope_append_kernel(
    Src src, const __nv_bfloat16* __restrict__ bias, const int* __restrict__ row_slot,
    const int* __restrict__ pos_by_slot, const int* __restrict__ row_pos, const int* __restrict__ page_table,
    int max_pages,
    const float* __restrict__ cos_t, const float* __restrict__ sin_t, int B, int nq, int nkv, int D, int P,
    __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache) {
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrQkvRope);
  pdl_wait();
  trace_mark(trs, 2);
  const int heads = nq + nkv;
  const int half = D / 2;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < (long long)B * heads * half) {
    const int b = (int)(t / (heads * half));
    const int rem = (int)(t - (long long)b * heads * half);
    const int h = rem / half, i = rem % half;
    const int slot = row_slot[b];
    const long long N = (long long)(nq + 2 * nkv) * D;
    const int pos = slot >= 0 ? (row_pos ? row_pos[b] : pos_by_slot[slot]) : 0;
    const long long rowoff = (long long)b * N;
    const float cs = cos_t[(size_t)pos * half + i];
    const float sn = sin_t[(size_t)pos * half + i];
    if (h < nq) {
      const int c0 = h * D;
      const long long off[2] = {rowoff + c0 + i, rowoff + c0 + i + half};
      float x[2];
      src_sum_multi<2>(src, off, x);
      if (bias) { x[0] += bf2f(bias[c0 + i]); x[1] += bf2f(bias[c0 + i + half]); }
      __nv_bfloat16* q = q_out + ((size_t)b * nq + h) * D;
      q[i] = f2bf(x[0] * cs - x[1] * sn);
      q[i + half] = f2bf(x[1] * cs + x[0] * sn);
    } else if (slot >= 0) {
      const int j = h - nq;
      const int kc0 = nq * D + j * D;
      const int vc0 = (nq + nkv) * D + j * D;
      const int page = page_table[(size_t)slot * max_pages + pos / P];
      const long long off[4] = {rowoff + kc0 + i, rowoff + kc0 + i + half, rowoff + vc0 + i, rowoff + vc0 + i + half};
      float x[4];
      src_sum_multi<4>(src, off, x);
      if (bias) {
        x[0] += bf2f(bias[kc0 + i]); x[1] += bf2f(bias[kc0 + i + half]);
        x[2] += bf2f(bias[vc0 + i]); x[3] += bf2f(bias[vc0 + i + half]);
      }
      const size_t off_c = (((size_t)page * nkv + j) * P + (pos % P)) * D;
      k_cache[off_c + i] = f2bf(x[0] * cs - x[1] * sn);
      k_cache[off_c + i + half] = f2bf(x[1] * cs + x[0] * sn);
      v_cache[off_c + i] = f2bf(x[2]);
      v_cache[off_c + i + half] = f2bf(x[3]);
    }
  }
  trace_mark(trs, 3);
}

// ------------------------------------------------------------- SiLU * up ---
// partial layout [split][B][2F] = [gate rows | up rows]; out[b][f] = bf16(silu(g) * u)
__global__ void silu_mul_kernel(Src src, int B, int F, __nv_bfloat16* __restrict__ out, int ldo) {
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrSilu);
  pdl_wait();
  trace_mark(trs, 2);
  const int F4 = F / 4;
  const long long total = (long long)B * F4;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(t / F4), f4 = (int)(t % F4);
    const long long row4 = (long long)b * 2 * F4;
    // interleaved 64-row blocks [gate c | up c]: 16 float4 per half-block
    const long long g4 = (f4 / 16) * 32 + (f4 % 16);
    const float4 g = src_sum4(src, row4 + g4);
    const float4 u = src_sum4(src, row4 + g4 + 16);
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + (size_t)b * ldo) + 2 * f4;
    o[0] = __floats2bfloat162_rn(g.x / (1.f + __expf(-g.x)) * u.x, g.y / (1.f + __expf(-g.y)) * u.y);
    o[1] = __floats2bfloat162_rn(g.z / (1.f + __expf(-g.z)) * u.z, g.w / (1.f + __expf(-g.w)) * u.w);
  }
  trace_mark(trs, 3);
}

// ------------------------------------------------------- greedy argmax ---
// Stage 1: per (row, vocab chunk) max with the smallest index on ties.
constexpr int kArgmaxThreads = 256;
__device__ __forceinline__ void cand_merge(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__global__ void __launch_bounds__(kArgmaxThreads) argmax_stage1_kernel(Src src, int B, int V, int vocab_offset,
                                                                      int nchunk, ArgmaxCand* __restrict__ cand,
                                                                      SignalSpec sig, SamplerSpec smp) {
  __shared__ float sv[kArgmaxThreads / 32];
  __shared__ int si[kArgmaxThreads / 32];
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrArgmax1);
  pdl_wait();
  trace_mark(trs, 2);
  const int b = blockIdx.x, c = blockIdx.y;
  const int per = ((V + nchunk - 1) / nchunk + 3) & ~3;
  const int lo = c * per, hi = min(V, lo + per);
  float best = -INFINITY;
  int bidx = 0x7fffffff;
  if (smp.seeds != nullptr) {
    // stochastic: logit / T + Gumbel(philox(ctr = (pos + 1, global vocab index), key = seed))
    const int slot = smp.row_slot[b];
    const uint64_t key = slot >= 0 ? smp.seeds[slot] : 0ull;
    const uint32_t pnext =
        slot >= 0 ? (uint32_t)((smp.row_pos ? smp.row_pos[b] : smp.pos_by_slot[slot]) + 1) : 0u;
    const uint2 k = make_uint2((uint32_t)key, (uint32_t)(key >> 32));
    for (int j = lo + threadIdx.x; j < hi; j += kArgmaxThreads) {
      const int gv = j + vocab_offset;
      const uint4 r = philox4x32_10(make_uint4(pnext, (uint32_t)gv, 0u, 0u), k);
      cand_merge(best, bidx, src_sum(src, (long long)b * V + j) * smp.inv_temp + gumbel_of(r.x), gv);
    }
  } else if ((V & 3) == 0) {
    for (int j = lo + 4 * threadIdx.x; j < hi; j += 4 * kArgmaxThreads) {
      const float4 v = src_sum4(src, ((long long)b * V + j) / 4);
      cand_merge(best, bidx, v.x, j + vocab_offset);
      cand_merge(best, bidx, v.y, j + 1 + vocab_offset);
      cand_merge(best, bidx, v.z, j + 2 + vocab_offset);
      cand_merge(best, bidx, v.w, j + 3 + vocab_offset);
    }
  } else {
    for (int j = lo + threadIdx.x; j < hi; j += kArgmaxThreads)
      cand_merge(best, bidx, src_sum(src, (long long)b * V + j), j + vocab_offset);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
    cand_merge(best, bidx, v2, i2);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = best;
    si[w] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kArgmaxThreads / 32; ++k) cand_merge(best, bidx, sv[k], si[k]);
    cand[(size_t)b * nchunk + c] = ArgmaxCand{best, bidx};
  }
  do_signal(sig);
  trace_mark(trs, 3);
}

// Stage 2: reduce the candidates of every TP rank (list order = rank order),
// append the token to the sample's history and advance its position.
__global__ void argmax_finalize_kernel(CandList cands, int nchunk, WaitSpec wait, const int* __restrict__ row_slot,
                                       int* __restrict__ pos_by_slot, const int* __restrict__ prompt_len,
                                       int* __restrict__ history, int hist_ld, int* __restrict__ out_tok) {
  const int b = blockIdx.x;
  // the step's last kernel releases its dependents only after the new positions are written:
  // the next step's attention streams KV pages before its own wait, from these positions
  const unsigned int trs = trace_begin(kTrArgmax2);
  pdl_wait();
  do_wait(wait);
  trace_mark(trs, 2);
  float best = -INFINITY;
  int bidx = 0x7fffffff;
#pragma unroll 4
  for (int k = threadIdx.x; k < cands.n * nchunk; k += blockDim.x) {
    const ArgmaxCand c = cands.p[k / nchunk][(size_t)b * nchunk + (k % nchunk)];
    cand_merge(best, bidx, c.val, c.idx);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
    cand_merge(best, bidx, v2, i2);
  }
  if (blockDim.x > 32) {  // (many candidates per row: the LM-head epilogue's per-tile ones)
    __shared__ float s_v[32];
    __shared__ int s_i[32];
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      s_v[w] = best;
      s_i[w] = bidx;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 1; k < nw; ++k) cand_merge(best, bidx, s_v[k], s_i[k]);
  }
  if (threadIdx.x == 0) {
    if (out_tok) out_tok[b] = bidx;
    const int slot = row_slot[b];
    if (slot >= 0) {
      const int pos = pos_by_slot[slot];
      // prompt positions are teacher-forced (prefill through the decode path)
      if (prompt_len == nullptr || pos + 1 >= prompt_len[slot]) history[(size_t)slot * hist_ld + pos + 1] = bidx;
      pos_by_slot[slot] = pos + 1;
    }
  }
  __threadfence();
  pdl_launch_dependents();
  trace_mark(trs, 3);
}

__global__ void epoch_advance_kernel(uint64_t* epoch) {
  pdl_wait();  // (step boundary: dependents launch after the epoch moved, see argmax_finalize)
  *epoch += 1ull;
  __threadfence();
  pdl_launch_dependents();
}

// Plain fp32 sum of a Src into a dense buffer (tests / logits export).
__global__ void sum_src_kernel(Src src, long long n, float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = src_sum(src, i);
}

// -------------------------------------------------------------- launchers ---
static int grid_for(long long work, int per_block, int cap) {
  long long g = (work + per_block - 1) / per_block;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

int embed(const int* row_slot, const int* pos_by_slot, const int* row_pos, const int* history, int hist_ld,
          const void* table, int H, int B, float* resid, cudaStream_t st) {
  TPS_CHECK_ARG(H % 2 == 0 && B > 0, "embed: H must be even, B > 0");
  return launch_k(embed_kernel, dim3(B), dim3(256), 0, st, true, row_slot, pos_by_slot, row_pos, history, hist_ld,
                  reinterpret_cast<const __nv_bfloat16*>(table), H, resid);
}

static bool g_norm_cluster = [] {
  const char* e = getenv("TPS_NORM_CLUSTER");
  return !(e && e[0] == '0');
}();

int add_norm(float* resid, const Src& src, const WaitSpec& wait, const void* w, float eps, int H, int B,
             void* out, int ldo, cudaStream_t st) {
  // tail batches: spread each row over a cluster (measured: TP8 B=1 step 1.93 -> 1.58 ms); at
  // B >= 32 one 512-thread CTA per row is faster (TP1 B=64: 4.67 vs 4.95 ms)
  if (g_norm_cluster && B <= 16 && H % 4 == 0 && H / 4 <= kNormCluster * kNormCThreads * kNormCVec &&
      src.n <= 16 && ldo % 2 == 0 && B > 0 && (src.n == 0 || src.stride % 4 == 0))
    return launch_kc(add_norm_cluster_kernel<false>, dim3(kNormCluster, B), dim3(kNormCThreads), kNormCluster, st,
                     true, resid, src, wait, (const uint64_t*)nullptr, 0, 0LL, (const uint64_t*)nullptr, 0u, 0u,
                     (unsigned long long*)nullptr, 0ULL, reinterpret_cast<const __nv_bfloat16*>(w), eps, H,
                     reinterpret_cast<__nv_bfloat16*>(out), ldo);
  TPS_CHECK_ARG(H % 4 == 0 && ldo % 2 == 0 && B > 0, "add_norm: H must be a multiple of 4");
  TPS_CHECK_ARG(H / 4 <= kNormThreads * kNormVec, "add_norm: H > 8192");
  TPS_CHECK_ARG(src.n == 0 || src.stride % 4 == 0, "add_norm: source stride must be a multiple of 4");
  // a fused TP allreduce hands over tp x splits (<= 16) partials: one 16-wide load batch
  if (src.n > 8)
    return launch_k(add_norm_kernel<16>, dim3(B), dim3(kNormThreads), 0, st, true, resid, src, wait,
                    reinterpret_cast<const __nv_bfloat16*>(w), eps, H, reinterpret_cast<__nv_bfloat16*>(out), ldo);
  return launch_k(add_norm_kernel<8>, dim3(B), dim3(kNormThreads), 0, st, true, resid, src, wait,
                  reinterpret_cast<const __nv_bfloat16*>(w), eps, H, reinterpret_cast<__nv_bfloat16*>(out), ldo);
}

int add_norm_ll(float* resid, const uint64_t* ll, int nsrc, long long stride, const uint64_t* epoch, uint32_t mult,
                uint32_t add, const void* w, float eps, int H, int B, void* out, int ldo, uint64_t* ctr,
                uint64_t bump, cudaStream_t st) {
  TPS_CHECK_ARG(H % 4 == 0 && ldo % 2 == 0 && B > 0 && nsrc >= 1 && ll && epoch, "add_norm_ll: bad arguments");
  TPS_CHECK_ARG(H / 4 <= kNormThreads * kNormVec, "add_norm_ll: H > 8192");
  TPS_CHECK_ARG(stride % 4 == 0 && (reinterpret_cast<uintptr_t>(ll) & 15) == 0, "add_norm_ll: 16B-aligned slots");
  if (g_norm_cluster && H / 4 <= kNormCluster * kNormCThreads * kNormCVec) {
    Src none{nullptr, 0, 0};
    WaitSpec nowait{nullptr, nullptr, 0, 0};
    return launch_kc(add_norm_cluster_kernel<true>, dim3(kNormCluster, B), dim3(kNormCThreads), kNormCluster, st,
                     true, resid, none, nowait, ll, nsrc, (long long)stride, epoch, mult, add,
                     reinterpret_cast<unsigned long long*>(ctr), (unsigned long long)bump,
                     reinterpret_cast<const __nv_bfloat16*>(w), eps, H, reinterpret_cast<__nv_bfloat16*>(out), ldo);
  }
  return launch_k(add_norm_ll_kernel, dim3(B), dim3(kNormThreads), 0, st, true, resid, ll, nsrc, stride, epoch,
                  mult, add, reinterpret_cast<const __nv_bfloat16*>(w), eps, H,
                  reinterpret_cast<__nv_bfloat16*>(out), ldo, reinterpret_cast<unsigned long long*>(ctr),
                  (unsigned long long)bump);
}

int reduce_push(const Src& src, const DstList& dst, long long n, const SignalSpec& sig, cudaStream_t st) {
  TPS_CHECK_ARG(n % 4 == 0 && src.n >= 1 && dst.n >= 1 && src.stride % 4 == 0,
                "reduce_push: n % 4 == 0, >=1 src/dst");
  return launch_k(reduce_push_kernel, dim3(kPushBlocks), dim3(256), 0, st, true, src, dst, n / 4, sig);
}

int reduce_push_ll(const Src& src, const DstList& dst, long long n, const uint64_t* epoch, uint32_t mult,
                   uint32_t add, cudaStream_t st) {
  TPS_CHECK_ARG(n % 4 == 0 && src.n >= 1 && dst.n >= 1 && src.stride % 4 == 0 && epoch,
                "reduce_push_ll: n % 4 == 0, >=1 src/dst, epoch");
  const long long n4 = n / 4;
  const int grid = (int)std::min<long long>(4LL * kNumSMs, (n4 + 255) / 256);
  return launch_k(reduce_push_ll_kernel, dim3(grid > 0 ? grid : 1), dim3(256), 0, st, true, src, dst, n4, epoch,
                  mult, add);
}

int qkv_rope_append(const Src& src, const void* bias, const int* row_slot, const int* pos_by_slot,
                    const int* row_pos, const int* page_table, int max_pages, const float* cos_t,
                    const float* sin_t, int B, int nq,
                    int nkv, int D, int P, void* q_out, void* k_cache, void* v_cache, cudaStream_t st) {
  TPS_CHECK_ARG(D % 2 == 0 && D <= 256 && B > 0 && nq > 0 && nkv > 0, "qkv_rope_append: bad shape");
  const long long threads = (long long)B * (nq + nkv) * (D / 2);
  return launch_k(qkv_rope_append_kernel, dim3((unsigned)((threads + 127) / 128)), dim3(128), 0, st, true, src,
                  reinterpret_cast<const __nv_bfloat16*>(bias), row_slot, pos_by_slot, row_pos, page_table,
                  max_pages,
                  cos_t, sin_t, B, nq, nkv, D, P, reinterpret_cast<__nv_bfloat16*>(q_out),
                  reinterpret_cast<__nv_bfloat16*>(k_cache), reinterpret_cast<__nv_bfloat16*>(v_cache));
}

int silu_mul(const Src& src, int B, int F, void* out, int ldo, cudaStream_t st) {
  TPS_CHECK_ARG(B > 0 && F > 0 && F % 4 == 0 && ldo % 4 == 0 && src.stride % 4 == 0,
                "silu_mul: F, ldo must be multiples of 4");
  const long long total = (long long)B * (F / 4);
  return launch_k(silu_mul_kernel, dim3(grid_for(total, 128, 4 * kNumSMs)), dim3(128), 0, st, true, src, B, F,
                  reinterpret_cast<__nv_bfloat16*>(out), ldo);
}

int argmax_stage1(const Src& src, int B, int V, int vocab_offset, int nchunk, void* cand, const SignalSpec& sig,
                  cudaStream_t st, const SamplerSpec* smp) {
  TPS_CHECK_ARG(B > 0 && V > 0 && nchunk > 0, "argmax_stage1: bad shape");
  SamplerSpec greedy{nullptr, nullptr, nullptr, nullptr, 1.f};
  return launch_k(argmax_stage1_kernel, dim3(B, nchunk), dim3(kArgmaxThreads), 0, st, true, src, B, V,
                  vocab_offset, nchunk, reinterpret_cast<ArgmaxCand*>(cand), sig, smp ? *smp : greedy);
}

int argmax_finalize(const CandList& cands, int nchunk, const WaitSpec& wait, int B, const int* row_slot,
                    int* pos_by_slot, const int* prompt_len, int* history, int hist_ld, int* out_tok,
                    cudaStream_t st) {
  TPS_CHECK_ARG(B > 0 && cands.n >= 1 && cands.n <= kMaxPeers, "argmax_finalize: bad args");
  const int threads = cands.n * nchunk > 256 ? 256 : 32;
  return launch_k(argmax_finalize_kernel, dim3(B), dim3(threads), 0, st, true, cands, nchunk, wait, row_slot,
                  pos_by_slot, prompt_len, history, hist_ld, out_tok);
}

int epoch_advance(uint64_t* epoch, cudaStream_t st) {
  return launch_k(epoch_advance_kernel, dim3(1), dim3(1), 0, st, true, epoch);
}

int sum_src(const Src& src, long long n, float* out, cudaStream_t st) {
  return launch_k(sum_src_kernel, dim3(grid_for(n, 256, 4 * kNumSMs)), dim3(256), 0, st, false, src, n, out);
}

int trace_register_decode(uint64_t* p, unsigned int* c, unsigned int n) { return trace_register(p, c, n); }

int configure_decode_ops() {
  TPS_MAX_CARVEOUT(embed_kernel);
  TPS_MAX_CARVEOUT(add_norm_kernel<8>);
  TPS_MAX_CARVEOUT(add_norm_kernel<16>);
  TPS_MAX_CARVEOUT(add_norm_ll_kernel);
  TPS_MAX_CARVEOUT(add_norm_cluster_kernel<false>);
  TPS_MAX_CARVEOUT(add_norm_cluster_kernel<true>);
  TPS_MAX_CARVEOUT(reduce_push_kernel);
  TPS_MAX_CARVEOUT(reduce_push_ll_kernel);
  TPS_MAX_CARVEOUT(qkv_rope_append_kernel);
  TPS_MAX_CARVEOUT(silu_mul_kernel);
  TPS_MAX_CARVEOUT(argmax_stage1_kernel);
  TPS_MAX_CARVEOUT(argmax_finalize_kernel);
  TPS_MAX_CARVEOUT(epoch_advance_kernel);
  TPS_MAX_CARVEOUT(sum_src_kernel);
  return kOk;
}

}  // namespace tps
