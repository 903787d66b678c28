#include <stdlib.h>
// Paged GQA decode attention (flash-decoding split-KV with in-kernel merge), sm_100a.
//
// The reference prices this work as the KV term of oracle_decode_latency,
// t * kv_bytes_per_token / (tp * hbm_bw) (tpshift/latency.py:123): one pass over
// every live token's K and V head slice. The kernel is HBM-bound, so it is built
// around the page stream:
//   * KV layout per layer is [page][kv_head][64 tokens][D] bf16, so one
//     (page, kv-head) slice is a contiguous 16 KB chunk (D=128). The same chunk
//     is the unit the Switch Executor migrates.
//   * grid = (kv_head, row, split): long contexts are split across CTAs (>= 2
//     pages each) so a tail batch of 1 still spreads over the 148 SMs; the
//     last CTA of a (row, kv_head) to finish merges the splits' (max, sum, O)
//     states with the max-rescaled log-sum-exp and writes the bf16 output --
//     no separate combine launch.
//   * 3-stage cp.async ring into an XOR-swizzled smem tile (conflict-free
//     fragment loads); the G query heads sharing a KV head form the 16-row
//     MMA operand, so QK^T and PV run on the tensor pipe and the CTA only
//     streams bytes.
#include <cooperative_groups.h>

#include "attention_common.cuh"

namespace tps {

constexpr int kMinPagesPerSplit = 2;
constexpr int kMaxAttnSplits = 128;
int attn_fixed_splits(int B, int nkv, int max_pages);

// TMA = true: pages arrive as four SWIZZLE_128B tensor-map boxes (K/V x two 64-column halves)
// issued by one thread and tracked by an mbarrier per ring stage, instead of 2 x 1024 16-byte
// cp.async per page from every thread (LSU-throttled at short contexts).
template <int D, bool TMA>
__global__ void __launch_bounds__(kAttnThreads) paged_attn_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __nv_bfloat16* __restrict__ v_cache, const int* __restrict__ row_slot,
    const int* __restrict__ pos_by_slot, const int* __restrict__ row_pos, const int* __restrict__ page_table,
    int max_pages, int nq, int nkv,
    int G, int nsplit, float scale_log2, float* __restrict__ part_m, float* __restrict__ part_l,
    float* __restrict__ part_o, unsigned int* __restrict__ merge_ctr, __nv_bfloat16* __restrict__ out,
    Src qkv, const __nv_bfloat16* __restrict__ qkv_bias, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, int early_ok, const __grid_constant__ CUtensorMap tmk,
    const __grid_constant__ CUtensorMap tmv) {
  constexpr int CPR = D / 8;       // 16-byte chunks per token row
  constexpr int TILE = kPage * D;  // elements per K (or V) page slice
  constexpr int HALF = D / 2;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem_base = TMA ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023))
                           : smem_raw;  // (SWIZZLE_128B boxes land on 1024-byte boundaries)
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem_base);
  __nv_bfloat16* sv = sk + kAttnStages * TILE;
  __shared__ int s_last;
  __shared__ __align__(8) uint64_t full_bar[kAttnStages];
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < kAttnStages; ++i) mbar_init(&full_bar[i], 1);
      fence_barrier_init();
    }
    __syncthreads();
  }
  // fused decode path: q (rotated) of this KV group and the current token's k/v,
  // finished here from the QKV projection's split partials (no separate rope kernel)
  __shared__ __align__(16) __nv_bfloat16 sq[16 * D];
  __shared__ __align__(16) __nv_bfloat16 skv[2 * D];
  const bool fused = qkv.n > 0;

  const int kvh = blockIdx.x, b = blockIdx.y, split = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, c = lane & 3;

  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrAttnSplit);
  // decode: the first pages stream before the programmatic wait (every cached token but the
  // current one was written by earlier steps; its row is refreshed after the wait, or -- fused
  // form -- patched in from the k/v this kernel finishes)
  const bool early = row_pos == nullptr && early_ok;
  if (!early) pdl_wait();
  trace_mark(trs, 2);

  const int slot = row_slot[b];
  const int ctx = slot >= 0 ? (row_pos ? row_pos[b] : pos_by_slot[slot]) + 1 : 0;
  const int npages = (ctx + kPage - 1) / kPage;
  int pps = (npages + nsplit - 1) / nsplit;
  if (pps < kMinPagesPerSplit) pps = kMinPagesPerSplit;
  const int active = (npages + pps - 1) / pps;
  const int p0 = split * pps;
  const int p1 = min(npages, p0 + pps);
  const int head0 = kvh * G;
  float* wm = reinterpret_cast<float*>(smem_raw);
  float* wl = wm + 4 * 16;
  float* wo = wl + 4 * 16;  // [warp][16][D]

  if (p0 >= p1) {
    if (early) pdl_wait();
    for (int h = tid; h < G; h += kAttnThreads) {
      const size_t base = ((size_t)b * nq + head0 + h) * nsplit + split;
      part_m[base] = -INFINITY;
      part_l[base] = 0.f;
    }
  } else {
    const int* pt = page_table + (size_t)slot * max_pages;
    auto load_page = [&](int p, int st) {
      if constexpr (TMA) {
        if (tid == 0) {
          const int row0 = (pt[p] * nkv + kvh) * kPage;
          const uint64_t pol = policy_evict_first();
          mbar_arrive_expect_tx(&full_bar[st], 2 * TILE * 2);
#pragma unroll
          for (int h = 0; h < D / 64; ++h) {
            tma_load_2d(sk + st * TILE + h * kPage * 64, &tmk, &full_bar[st], h * 64, row0, pol);
            tma_load_2d(sv + st * TILE + h * kPage * 64, &tmv, &full_bar[st], h * 64, row0, pol);
          }
        }
      } else {
        const size_t goff = ((size_t)pt[p] * nkv + kvh) * TILE;
        const __nv_bfloat16* gk = k_cache + goff;
        const __nv_bfloat16* gv = v_cache + goff;
        __nv_bfloat16* dk = sk + st * TILE;
        __nv_bfloat16* dv = sv + st * TILE;
#pragma unroll
        for (int i = tid; i < kPage * CPR; i += kAttnThreads) {
          const int row = i / CPR, cc = i % CPR;
          const int sw = row * D + ((cc ^ (row & 7)) * 8);
          cp_async16(dk + sw, gk + row * D + cc * 8);
          cp_async16(dv + sw, gv + row * D + cc * 8);
        }
      }
    };

#pragma unroll
    for (int i = 0; i < kAttnStages - 1; ++i) {
      if (p0 + i < p1) load_page(p0 + i, i);
      cp_async_commit();
    }
    if (early) pdl_wait();

    const bool owner = fused && (p1 == npages);  // this split holds the current token's page
    if (fused) {
      // sum split partials + bias, rotate-half RoPE at pos = ctx-1, round to bf16
      const int pos = ctx - 1;
      const long long N = (long long)(nq + 2 * nkv) * D;
      const long long row = (long long)b * N;
      auto val = [&](int col) {
        float v = qkv_bias ? bf2f(qkv_bias[col]) : 0.f;
        const float* p = qkv.base + row + col;
        for (int s = 0; s < qkv.n; ++s) v += p[(long long)s * qkv.stride];
        return v;
      };
      for (int i = tid; i < 16 * HALF; i += kAttnThreads) {
        const int h = i / HALF, d = i % HALF;
        float y1 = 0.f, y2 = 0.f;
        if (h < G) {
          const float cs = cos_t[(size_t)pos * HALF + d], sn = sin_t[(size_t)pos * HALF + d];
          const int c0 = (head0 + h) * D;
          const float x1 = val(c0 + d), x2 = val(c0 + d + HALF);
          y1 = x1 * cs - x2 * sn;
          y2 = x2 * cs + x1 * sn;
        }
        sq[h * D + d] = f2bf(y1);
        sq[h * D + d + HALF] = f2bf(y2);
      }
      if (owner) {
        const int page = pt[pos / kPage];
        const size_t off = (((size_t)page * nkv + kvh) * kPage + (pos % kPage)) * D;
        for (int i = tid; i < 2 * HALF; i += kAttnThreads) {
          const bool is_v = i >= HALF;
          const int d = i % HALF;
          const int c0 = (is_v ? (nq + nkv + kvh) : (nq + kvh)) * D;
          const float x1 = val(c0 + d), x2 = val(c0 + d + HALF);
          float y1 = x1, y2 = x2;
          if (!is_v) {
            const float cs = cos_t[(size_t)pos * HALF + d], sn = sin_t[(size_t)pos * HALF + d];
            y1 = x1 * cs - x2 * sn;
            y2 = x2 * cs + x1 * sn;
          }
          __nv_bfloat16* cache = const_cast<__nv_bfloat16*>(is_v ? v_cache : k_cache) + off;
          cache[d] = f2bf(y1);
          cache[d + HALF] = f2bf(y2);
          skv[(is_v ? D : 0) + d] = f2bf(y1);
          skv[(is_v ? D : 0) + d + HALF] = f2bf(y2);
        }
      }
      __syncthreads();
    }

    // Q fragments for the (up to 16) query heads of this KV group, held for the whole loop.
    uint32_t qa[D / 16][4];
    if (fused) {
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const int d0 = ks * 16 + 2 * c;
        qa[ks][0] = *reinterpret_cast<const uint32_t*>(sq + g * D + d0);
        qa[ks][1] = *reinterpret_cast<const uint32_t*>(sq + (g + 8) * D + d0);
        qa[ks][2] = *reinterpret_cast<const uint32_t*>(sq + g * D + d0 + 8);
        qa[ks][3] = *reinterpret_cast<const uint32_t*>(sq + (g + 8) * D + d0 + 8);
      }
    } else {
      load_q_frags<D>(qa, q + ((size_t)b * nq + head0) * D, G);
    }

    float m_r[2] = {-INFINITY, -INFINITY};
    float l_r[2] = {0.f, 0.f};
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

    for (int it = 0; p0 + it < p1; ++it) {
      const int st = it % kAttnStages;
      if constexpr (TMA) {
        __syncthreads();  // every warp is done with the stage the next load overwrites
        const int nxt = it + kAttnStages - 1;
        if (p0 + nxt < p1) {
          if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          load_page(p0 + nxt, nxt % kAttnStages);
        }
        mbar_wait(&full_bar[st], (uint32_t)((it / kAttnStages) & 1));
      } else {
        cp_async_wait<kAttnStages - 2>();
        __syncthreads();
        const int nxt = it + kAttnStages - 1;
        if (p0 + nxt < p1) load_page(p0 + nxt, nxt % kAttnStages);
        cp_async_commit();
      }
      if (early && !fused && it < kAttnStages - 1 && p0 + it == npages - 1) {
        // issued before the wait: refresh the current token's K/V row
        const int r = (ctx - 1) % kPage;
        const size_t goff = ((size_t)pt[p0 + it] * nkv + kvh) * TILE + (size_t)r * D;
        for (int i = tid; i < 2 * CPR; i += kAttnThreads) {
          const bool is_v = i >= CPR;
          const int cc = i % CPR;
          const uint4 v = __ldcg(reinterpret_cast<const uint4*>((is_v ? v_cache : k_cache) + goff) + cc);
          *reinterpret_cast<uint4*>((is_v ? sv : sk) + st * TILE + tile_off<D, TMA>(r, cc)) = v;
        }
        __syncthreads();
      }
      if (owner && p0 + it == npages - 1) {
        // the current token's k/v were computed in-kernel: patch them into the landed tile
        const int r = (ctx - 1) % kPage;
        for (int i = tid; i < 2 * CPR; i += kAttnThreads) {
          const bool is_v = i >= CPR;
          const int cc = i % CPR;
          __nv_bfloat16* dst = (is_v ? sv : sk) + st * TILE + tile_off<D, TMA>(r, cc);
          *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(skv + (is_v ? D : 0) + cc * 8);
        }
        __syncthreads();
      }
      attend_page<D, TMA>(sk + st * TILE, sv + st * TILE, qa, (p0 + it) * kPage, ctx, scale_log2, m_r, l_r, o);
    }
    cp_async_wait<0>();

#pragma unroll
    for (int r = 0; r < 2; ++r) {
      l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
      l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
    }

    // merge the 4 warps' partial softmax states through shared memory
    __syncthreads();
    if (c == 0) {
      wm[warp * 16 + g] = m_r[0];
      wm[warp * 16 + g + 8] = m_r[1];
      wl[warp * 16 + g] = l_r[0];
      wl[warp * 16 + g + 8] = l_r[1];
    }
#pragma unroll
    for (int dn = 0; dn < D / 8; ++dn) {
      const int d = dn * 8 + 2 * c;
      wo[(warp * 16 + g) * D + d] = o[dn][0];
      wo[(warp * 16 + g) * D + d + 1] = o[dn][1];
      wo[(warp * 16 + g + 8) * D + d] = o[dn][2];
      wo[(warp * 16 + g + 8) * D + d + 1] = o[dn][3];
    }
    __syncthreads();
    for (int i = tid; i < G * D; i += kAttnThreads) {
      const int h = i / D, d = i % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * 16 + h]);
      float L = 0.f, acc = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float mw = wm[w * 16 + h];
        const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
        L += wl[w * 16 + h] * f;
        acc += wo[(w * 16 + h) * D + d] * f;
      }
      const size_t base = ((size_t)b * nq + head0 + h) * nsplit + split;
      part_o[base * D + d] = acc;
      if (d == 0) {
        part_m[base] = M;
        part_l[base] = L;
      }
    }
  }

  // ---- split merge by the last CTA of this (row, kv head) ----
  // (with many splits the merge is done by attn_combine_kernel instead: merge_ctr == null)
  trace_mark(trs, 3);  // (a merging CTA overwrites this with its own exit below)
  if (merge_ctr == nullptr) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned int prev = atomicAdd(&merge_ctr[b * nkv + kvh], 1u);
    s_last = (prev == (unsigned int)nsplit - 1u);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  float* fac = wo + 4 * 16 * D;      // [16][kMaxAttnSplits]
  float* inv_l = fac + 16 * kMaxAttnSplits;  // [16]
  for (int h = warp; h < G; h += 4) {
    const size_t base = ((size_t)b * nq + head0 + h) * nsplit;
    float M = -INFINITY;
    for (int s2 = lane; s2 < active; s2 += 32) M = fmaxf(M, __ldcg(part_m + base + s2));
    M = warp_max(M);
    float L = 0.f;
    for (int s2 = lane; s2 < active; s2 += 32) {
      const float ms = __ldcg(part_m + base + s2);
      const float f = (ms == -INFINITY || M == -INFINITY) ? 0.f : exp2f(ms - M);
      fac[h * kMaxAttnSplits + s2] = f;
      L += __ldcg(part_l + base + s2) * f;
    }
    L = warp_sum(L);
    if (lane == 0) inv_l[h] = L > 0.f ? 1.f / L : 0.f;
  }
  __syncthreads();
  for (int i = tid; i < G * D; i += kAttnThreads) {
    const int h = i / D, d = i % D;
    const float* po = part_o + ((size_t)b * nq + head0 + h) * nsplit * D + d;
    const float* fh = fac + h * kMaxAttnSplits;
    float acc = 0.f;
    // independent loads in batches of 8: the merge is latency-, not bandwidth-bound
    for (int s0 = 0; s0 < active; s0 += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (s0 + j < active) ? __ldcg(po + (size_t)(s0 + j) * D) : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (s0 + j < active) acc += v[j] * fh[s0 + j];
    }
    out[((size_t)b * nq + head0 + h) * D + d] = f2bf(acc * inv_l[h]);
  }
  if (tid == 0) merge_ctr[b * nkv + kvh] = 0u;  // re-arm for the next launch / graph replay
  trace_mark(trs, 3);
}

// Many-split merge (long contexts at small batch): one CTA per (row, query head), one
// thread per head dim; the split maxima are reduced across lanes and every thread's
// partial-O loads are issued in batches of 16, so the merge costs ~one L2 round trip.
template <int D>
__global__ void __launch_bounds__(D) attn_combine_kernel(const int* __restrict__ row_slot,
                                                         const int* __restrict__ pos_by_slot,
                                                         const int* __restrict__ row_pos, int nq, int nsplit,
                                                         const float* __restrict__ part_m,
                                                         const float* __restrict__ part_l,
                                                         const float* __restrict__ part_o,
                                                         __nv_bfloat16* __restrict__ out) {
  __shared__ float fac[kMaxAttnSplits];
  __shared__ float s_inv;
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrAttnCombine);
  pdl_wait();
  trace_mark(trs, 2);
  const int b = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const int slot = row_slot[b];
  const int ctx = slot >= 0 ? (row_pos ? row_pos[b] : pos_by_slot[slot]) + 1 : 0;
  const int npages = (ctx + kPage - 1) / kPage;
  int pps = (npages + nsplit - 1) / nsplit;
  if (pps < kMinPagesPerSplit) pps = kMinPagesPerSplit;
  const int active = (npages + pps - 1) / pps;
  const size_t base = ((size_t)b * nq + h) * nsplit;
  if (d < 32) {
    float M = -INFINITY;
    for (int s = d; s < active; s += 32) M = fmaxf(M, part_m[base + s]);
    M = warp_max(M);
    float L = 0.f;
    for (int s = d; s < active; s += 32) {
      const float ms = part_m[base + s];
      const float f = (ms == -INFINITY || M == -INFINITY) ? 0.f : exp2f(ms - M);
      fac[s] = f;
      L += part_l[base + s] * f;
    }
    L = warp_sum(L);
    if (d == 0) s_inv = L > 0.f ? 1.f / L : 0.f;
  }
  __syncthreads();
  const float* po = part_o + base * D + d;
  float acc = 0.f;
  for (int s0 = 0; s0 < active; s0 += 16) {
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = (s0 + j < active) ? po[(size_t)(s0 + j) * D] : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (s0 + j < active) acc += v[j] * fac[s0 + j];
  }
  out[((size_t)b * nq + h) * D + d] = f2bf(acc * s_inv);
  trace_mark(trs, 3);
}

constexpr int kInKernelMergeMaxSplits = 4;

// ------------------------------------------------------------------------------------
// Tail-batch attention: one thread-block cluster per (row, kv head) segment. Each CTA of
// the cluster streams its slice of the segment's pages through the cp.async ring and keeps
// its (max, sum, O) softmax state in shared memory; after a cluster barrier every CTA merges
// a slice of the G x D output straight out of its peers' shared memory (DSMEM) -- no
// global partials, atomics or second kernel on the critical path of a 1..16-row step.
// (Round 1 had an opt-in variant streaming the first pages before the PDL wait, -3 % at TP8
// B=1; graph-replayed decode diverged from eager decode with it, root cause not found: the
// variant was removed in round 2. Every page is read after the wait.)

template <int D, bool TMA>
__global__ void __launch_bounds__(kAttnThreads) paged_attn_cluster_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __nv_bfloat16* __restrict__ v_cache, const int* __restrict__ row_slot,
    const int* __restrict__ pos_by_slot, const int* __restrict__ row_pos, const int* __restrict__ page_table,
    int max_pages, int nq, int nkv, int G, float scale_log2, __nv_bfloat16* __restrict__ out,
    const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv) {
  namespace cg = cooperative_groups;
  constexpr int CPR = D / 8;
  constexpr int TILE = kPage * D;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem_base = TMA ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023))
                           : smem_raw;
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem_base);
  __nv_bfloat16* sv = sk + kAttnStages * TILE;
  __shared__ __align__(8) uint64_t full_bar[kAttnStages];
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < kAttnStages; ++i) mbar_init(&full_bar[i], 1);
      fence_barrier_init();
    }
    __syncthreads();
  }
  __shared__ float c_m[16], c_l[16];
  __shared__ __align__(16) float c_o[16 * D];
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int seg = blockIdx.y;
  const int b = seg / nkv, kvh = seg % nkv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, c = lane & 3;
  pdl_launch_dependents();  // dependents may launch now: they read our outputs only after their own wait
  const unsigned int trs = trace_begin(kTrAttnSplit);
  pdl_wait();  // q and the current token's K/V row were written by the previous kernel
  const int slot = row_slot[b];
  const int ctx = slot >= 0 ? (row_pos ? row_pos[b] : pos_by_slot[slot]) + 1 : 0;
  const int npages = (ctx + kPage - 1) / kPage;
  const int pps = (npages + CL - 1) / CL;
  const int p0 = min(npages, crank * pps), p1 = min(npages, p0 + pps);
  const int head0 = kvh * G;
  float* wm = reinterpret_cast<float*>(smem_raw);
  float* wl = wm + 4 * 16;
  float* wo = wl + 4 * 16;  // [warp][16][D]
  float m_r[2] = {-INFINITY, -INFINITY};
  float l_r[2] = {0.f, 0.f};
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  if (p0 < p1) {
    const int* pt = page_table + (size_t)slot * max_pages;
    auto load_page = [&](int p, int st) {
      if constexpr (TMA) {
        if (tid == 0) {
          const int row0 = (pt[p] * nkv + kvh) * kPage;
          const uint64_t pol = policy_evict_first();
          mbar_arrive_expect_tx(&full_bar[st], 2 * TILE * 2);
#pragma unroll
          for (int h = 0; h < D / 64; ++h) {
            tma_load_2d(sk + st * TILE + h * kPage * 64, &tmk, &full_bar[st], h * 64, row0, pol);
            tma_load_2d(sv + st * TILE + h * kPage * 64, &tmv, &full_bar[st], h * 64, row0, pol);
          }
        }
      } else {
        const size_t goff = ((size_t)pt[p] * nkv + kvh) * TILE;
        const __nv_bfloat16* gk = k_cache + goff;
        const __nv_bfloat16* gv = v_cache + goff;
        __nv_bfloat16* dk = sk + st * TILE;
        __nv_bfloat16* dv = sv + st * TILE;
#pragma unroll
        for (int i = tid; i < kPage * CPR; i += kAttnThreads) {
          const int row = i / CPR, cc = i % CPR;
          const int sw = row * D + ((cc ^ (row & 7)) * 8);
          cp_async16(dk + sw, gk + row * D + cc * 8);
          cp_async16(dv + sw, gv + row * D + cc * 8);
        }
      }
    };
#pragma unroll
    for (int i = 0; i < kAttnStages - 1; ++i) {
      if (p0 + i < p1) load_page(p0 + i, i);
      cp_async_commit();
    }
    uint32_t qa[D / 16][4];
    load_q_frags<D>(qa, q + ((size_t)b * nq + head0) * D, G);
    for (int it = 0; p0 + it < p1; ++it) {
      const int st = it % kAttnStages;
      if constexpr (TMA) {
        __syncthreads();  // every warp is done with the stage the next load overwrites
        const int nxt = it + kAttnStages - 1;
        if (p0 + nxt < p1) {
          if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          load_page(p0 + nxt, nxt % kAttnStages);
        }
        mbar_wait(&full_bar[st], (uint32_t)((it / kAttnStages) & 1));
      } else {
        cp_async_wait<kAttnStages - 2>();
        __syncthreads();
        const int nxt = it + kAttnStages - 1;
        if (p0 + nxt < p1) load_page(p0 + nxt, nxt % kAttnStages);
        cp_async_commit();
      }
      attend_page<D, TMA>(sk + st * TILE, sv + st * TILE, qa, (p0 + it) * kPage, ctx, scale_log2, m_r, l_r, o);
    }
    cp_async_wait<0>();
  }
  trace_mark(trs, 2);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  // the CTA's own state: merge its 4 warps (as the split kernel does)
  __syncthreads();
  if (c == 0) {
    wm[warp * 16 + g] = m_r[0];
    wm[warp * 16 + g + 8] = m_r[1];
    wl[warp * 16 + g] = l_r[0];
    wl[warp * 16 + g + 8] = l_r[1];
  }
#pragma unroll
  for (int dn = 0; dn < D / 8; ++dn) {
    const int d = dn * 8 + 2 * c;
    wo[(warp * 16 + g) * D + d] = o[dn][0];
    wo[(warp * 16 + g) * D + d + 1] = o[dn][1];
    wo[(warp * 16 + g + 8) * D + d] = o[dn][2];
    wo[(warp * 16 + g + 8) * D + d + 1] = o[dn][3];
  }
  __syncthreads();
  for (int i = tid; i < G * D; i += kAttnThreads) {
    const int h = i / D, d = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * 16 + h]);
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = wm[w * 16 + h];
      const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      L += wl[w * 16 + h] * f;
      acc += wo[(w * 16 + h) * D + d] * f;
    }
    c_o[h * D + d] = acc;
    if (d == 0) {
      c_m[h] = M;
      c_l[h] = L;
    }
  }
  cluster.sync();
  // merge across the cluster. (1) every peer's (max, sum) per head, fetched in parallel
  // (thread t reads peer t / 16, head t % 16) -> per-(peer, head) rescale factors in smem;
  // (2) CTA r finishes output elements r, r + CL, ... of the G x D tile with all CL remote
  // loads of an element issued together (DSMEM latency is paid once, not CL times)
  __shared__ float s_pm[16 * 16], s_pl[16 * 16], s_f[16 * 16], s_inv[16];
  for (int t = tid; t < CL * 16; t += kAttnThreads) {
    const int r = t >> 4, h = t & 15;
    s_pm[t] = h < G ? *cluster.map_shared_rank(&c_m[h], r) : -INFINITY;
    s_pl[t] = h < G ? *cluster.map_shared_rank(&c_l[h], r) : 0.f;
  }
  __syncthreads();
  if (tid < 16) {
    const int h = tid;
    float M = -INFINITY;
    for (int r = 0; r < CL; ++r) M = fmaxf(M, s_pm[r * 16 + h]);
    float L = 0.f;
    for (int r = 0; r < CL; ++r) {
      const float mr = s_pm[r * 16 + h];
      const float f = (mr == -INFINITY || M == -INFINITY) ? 0.f : exp2f(mr - M);
      s_f[r * 16 + h] = f;
      L += s_pl[r * 16 + h] * f;
    }
    s_inv[h] = L > 0.f ? 1.f / L : 0.f;
  }
  __syncthreads();
  for (int i = crank * kAttnThreads + tid; i < G * D; i += CL * kAttnThreads) {
    const int h = i / D, d = i % D;
    float v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = r < CL ? *cluster.map_shared_rank(&c_o[h * D + d], r) : 0.f;
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r < CL) acc += v[r] * s_f[r * 16 + h];
    out[((size_t)b * nq + head0 + h) * D + d] = f2bf(acc * s_inv[h]);
  }
  cluster.sync();  // peers may still be reading this CTA's state
  trace_mark(trs, 3);
}

template <int D>
static constexpr int attn_smem() {
  return 2 * kAttnStages * kPage * D * 2;
}

int paged_attention_balanced(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                             const int* pos_by_slot, const int* row_pos, const int* page_table, int max_pages,
                             int B, int nq, int nkv, int D, float* part_m, float* part_l, float* part_o,
                             unsigned int* merge_ctr, void* out, cudaStream_t st);
int configure_attention_balanced();
int configure_attention_prefill();

int configure_attention() {
  int rc = configure_attention_balanced();
  if (!rc) rc = configure_attention_prefill();
  if (rc) return rc;
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_kernel<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    attn_smem<128>()));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_kernel<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    attn_smem<64>()));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    attn_smem<128>() + 1024));
  TPS_MAX_CARVEOUT((paged_attn_kernel<128, true>));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_cluster_kernel<128, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, attn_smem<128>()));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_cluster_kernel<64, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, attn_smem<64>()));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_cluster_kernel<128, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, attn_smem<128>() + 1024));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_cluster_kernel<128, false>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_cluster_kernel<64, false>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_cluster_kernel<128, true>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  TPS_MAX_CARVEOUT((paged_attn_cluster_kernel<128, false>));
  TPS_MAX_CARVEOUT((paged_attn_cluster_kernel<64, false>));
  TPS_MAX_CARVEOUT((paged_attn_cluster_kernel<128, true>));
  TPS_MAX_CARVEOUT((paged_attn_kernel<128, false>));
  TPS_MAX_CARVEOUT((paged_attn_kernel<64, false>));
  TPS_MAX_CARVEOUT(attn_combine_kernel<128>);
  TPS_MAX_CARVEOUT(attn_combine_kernel<64>);
  return kOk;
}

// Split policy: 0 = page-balanced schedule (when the (row, kv head) segments alone
// give a few hundred units of parallel work), else the fixed split count that
// keeps the grid within one wave of resident CTAs (2 per SM).
// TPS_ATTN_MIN_BAL=<n>: use the page-balanced schedule from B * nkv >= n (default 64)
static int g_min_bal = [] {
  const char* e = getenv("TPS_ATTN_MIN_BAL");
  return e ? atoi(e) : 64;
}();

// TPS_ATTN_EARLY=0: no KV streaming before the programmatic wait (A/B and debugging)
static int g_attn_early = [] {
  const char* e = getenv("TPS_ATTN_EARLY");
  return e ? atoi(e) : 1;
}();

// TPS_ATTN_MAX_CLUSTER=<n>: the cluster form for B * nkv <= n segments (default 8, 0 = off;
// measured at ctx 3072: TP8 B=8 1.55 vs 1.70 ms balanced; B*nkv = 16 is faster split/balanced)
static int g_max_cluster = [] {
  const char* e = getenv("TPS_ATTN_MAX_CLUSTER");
  return e ? atoi(e) : 8;
}();

// TPS_ATTN_CLUSTER_SIZE=<n>: CTAs per segment of the cluster form (default 16; 2..16)
static int g_cluster_size = [] {
  const char* e = getenv("TPS_ATTN_CLUSTER_SIZE");
  const int v = e ? atoi(e) : 16;
  return v < 2 ? 2 : (v > 16 ? 16 : v);
}();

// TPS_ATTN_TMA=0: the fixed-split decode attention stages its pages with cp.async instead of
// tensor-map TMA boxes (TMA measured: TP1 B=64 step 4.474 -> 4.432 ms at ctx 2048, 3.661 ->
// 3.644 at ctx 512; no LSU throttling of 2 x 1024 cp.async per page)
static int g_attn_tma = [] {
  const char* e = getenv("TPS_ATTN_TMA");
  return e ? atoi(e) : 1;
}();

int make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

// TPS_ATTN_TMA_CLUSTER=0: the cluster form stages its pages with cp.async instead of TMA boxes
// (TMA measured: TP8 B=1 ctx 2048 1.321 -> 1.299 ms, ctx 8192 1.518 -> 1.460; TP4 B=8 1.742 -> 1.700)
static int g_attn_tma_cluster = [] {
  const char* e = getenv("TPS_ATTN_TMA_CLUSTER");
  return e ? atoi(e) : 1;
}();

int attn_splits(int B, int nkv, int max_pages) {
  // page-balanced when the (row, kv head) segments give enough parallel work, and for a
  // single local KV head (TP-sharded GQA tail: measured faster than split + combine)
  if (B * nkv <= g_max_cluster) return -1;  // tail: one CTA cluster per (row, kv head)
  // one wave of fixed splits when it fills >= 80 % of the resident CTA slots (measured: bench
  // stage -1.4 % vs balanced at B = 16..64; one local KV head (TP4/TP8 Qwen2.5-7B) B = 12..64
  // -9..11 % per step); else, with more segments than slots, the page-balanced schedule
  if (B * nkv <= 2 * kNumSMs && g_min_bal == 64) {
    const int ns = attn_fixed_splits(B, nkv, max_pages);
    if ((long long)B * nkv * ns * 10 >= 8LL * 2 * kNumSMs) return ns;
  }
  if ((B * nkv >= g_min_bal || nkv == 1) && B <= kBalMaxRows) return 0;
  return attn_fixed_splits(B, nkv, max_pages);
}

int attn_fixed_splits(int B, int nkv, int max_pages) {
  int want = (2 * kNumSMs) / (B * nkv);
  const int cap = (max_pages + kMinPagesPerSplit - 1) / kMinPagesPerSplit;
  if (want > cap) want = cap;
  if (want > 32) want = 32;  // the last-CTA merge reads active x G x D partials: keep it short
  if (want < 1) want = 1;
  return want;
}

int paged_attention(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                    const int* pos_by_slot, const int* row_pos, const int* page_table, int max_pages,
                    int B, int nq, int nkv, int D,
                    int nsplit, float* part_m, float* part_l, float* part_o, unsigned int* merge_ctr, void* out,
                    const Src& qkv, const void* qkv_bias, const float* cos_t, const float* sin_t,
                    cudaStream_t st) {
  TPS_CHECK_ARG(B > 0 && nkv > 0 && nq % nkv == 0, "paged_attention: nq must be a multiple of nkv");
  TPS_CHECK_ARG(qkv.n == 0 || (cos_t && sin_t && !row_pos),
                "paged_attention: fused QKV finishing needs rope tables and is decode-only (row_pos == NULL)");
  const auto* bias = reinterpret_cast<const __nv_bfloat16*>(qkv_bias);
  const int G = nq / nkv;
  TPS_CHECK_ARG(G <= 16, "paged_attention: at most 16 query heads per KV head");
  TPS_CHECK_ARG(nsplit >= -1 && nsplit <= kMaxAttnSplits, "paged_attention: -1 <= nsplit <= 128");
  TPS_CHECK_ARG(nsplit > 0 || qkv.n == 0, "paged_attention: the fused QKV form needs an explicit split count");
  TPS_CHECK_ARG(nsplit >= 0 || B * nkv <= 65535, "paged_attention: too many segments for the cluster form");
  if (nsplit < 0) {
    // cluster kernel (tail batches): 16 CTAs per segment when there are few segments
    const int cl = g_cluster_size;  // (non-portable size 16: 16 CTAs of <= 2 per SM per cluster)
    const float scale = 1.4426950408889634f / sqrtf((float)D);
    const auto* qq = reinterpret_cast<const __nv_bfloat16*>(q);
    const auto* kk = reinterpret_cast<const __nv_bfloat16*>(k_cache);
    const auto* vv = reinterpret_cast<const __nv_bfloat16*>(v_cache);
    auto* oo = reinterpret_cast<__nv_bfloat16*>(out);
    CUtensorMap tmk{}, tmv{};
    if (D == 128 && g_attn_tma_cluster) {
      int rc = make_tmap_bf16(&tmk, k_cache, 1LL << 28, D, D, kPage);
      if (!rc) rc = make_tmap_bf16(&tmv, v_cache, 1LL << 28, D, D, kPage);
      if (rc) return rc;
      return launch_kcs(paged_attn_cluster_kernel<128, true>, dim3(cl, B * nkv), dim3(kAttnThreads), cl,
                        attn_smem<128>() + 1024, st, true, qq, kk, vv, row_slot, pos_by_slot, row_pos, page_table,
                        max_pages, nq, nkv, G, scale, oo, tmk, tmv);
    }
    if (D == 128)
      return launch_kcs(paged_attn_cluster_kernel<128, false>, dim3(cl, B * nkv), dim3(kAttnThreads), cl,
                        attn_smem<128>(), st, true, qq, kk, vv, row_slot, pos_by_slot, row_pos, page_table,
                        max_pages, nq, nkv, G, scale, oo, tmk, tmv);
    if (D == 64)
      return launch_kcs(paged_attn_cluster_kernel<64, false>, dim3(cl, B * nkv), dim3(kAttnThreads), cl,
                        attn_smem<64>(), st, true, qq, kk, vv, row_slot, pos_by_slot, row_pos, page_table,
                        max_pages, nq, nkv, G, scale, oo, tmk, tmv);
    return fail(kInvalid, "paged_attention: head_dim must be 64 or 128");
  }
  if (nsplit == 0)
    return paged_attention_balanced(q, k_cache, v_cache, row_slot, pos_by_slot, row_pos, page_table, max_pages, B,
                                    nq, nkv, D, part_m, part_l, part_o, merge_ctr, out, st);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  const dim3 grid(nkv, B, nsplit);
  const auto* qq = reinterpret_cast<const __nv_bfloat16*>(q);
  const auto* kk = reinterpret_cast<const __nv_bfloat16*>(k_cache);
  const auto* vv = reinterpret_cast<const __nv_bfloat16*>(v_cache);
  auto* oo = reinterpret_cast<__nv_bfloat16*>(out);
  const bool in_kernel = nsplit <= kInKernelMergeMaxSplits;
  unsigned int* mc = in_kernel ? merge_ctr : nullptr;
  int rc;
  CUtensorMap tmk{}, tmv{};
  const bool tma = g_attn_tma && D == 128 && qkv.n == 0;
  if (tma) {
    // the pool as a 2-D [rows][D] bf16 tensor, one (page, kv head) slice = 64 rows; a generous
    // row bound (boxes are only ever requested inside allocated pages)
    rc = make_tmap_bf16(&tmk, k_cache, 1LL << 28, D, D, kPage);
    if (!rc) rc = make_tmap_bf16(&tmv, v_cache, 1LL << 28, D, D, kPage);
    if (rc) return rc;
  }
  if (D == 128 && tma)
    rc = launch_k(paged_attn_kernel<128, true>, grid, dim3(kAttnThreads), attn_smem<128>() + 1024, st, true, qq, kk,
                  vv, row_slot, pos_by_slot, row_pos, page_table, max_pages, nq, nkv, G, nsplit, scale_log2, part_m,
                  part_l, part_o, mc, oo, qkv, bias, cos_t, sin_t, g_attn_early, tmk, tmv);
  else if (D == 128)
    rc = launch_k(paged_attn_kernel<128, false>, grid, dim3(kAttnThreads), attn_smem<128>(), st, true, qq, kk, vv,
                  row_slot, pos_by_slot, row_pos, page_table, max_pages, nq, nkv, G, nsplit, scale_log2, part_m,
                  part_l, part_o, mc, oo, qkv, bias, cos_t, sin_t, g_attn_early, tmk, tmv);
  else if (D == 64)
    rc = launch_k(paged_attn_kernel<64, false>, grid, dim3(kAttnThreads), attn_smem<64>(), st, true, qq, kk, vv,
                  row_slot, pos_by_slot, row_pos, page_table, max_pages, nq, nkv, G, nsplit, scale_log2, part_m,
                  part_l, part_o, mc, oo, qkv, bias, cos_t, sin_t, g_attn_early, tmk, tmv);
  else
    return fail(kInvalid, "paged_attention: head_dim must be 64 or 128");
  if (rc || in_kernel) return rc;
  if (D == 128)
    return launch_k(attn_combine_kernel<128>, dim3(B, nq), dim3(128), 0, st, true, row_slot, pos_by_slot, row_pos,
                    nq, nsplit, (const float*)part_m, (const float*)part_l, (const float*)part_o, oo);
  return launch_k(attn_combine_kernel<64>, dim3(B, nq), dim3(64), 0, st, true, row_slot, pos_by_slot, row_pos, nq,
                  nsplit, (const float*)part_m, (const float*)part_l, (const float*)part_o, oo);
}

int trace_register_attention(uint64_t* p, unsigned int* c, unsigned int n) { return trace_register(p, c, n); }

}  // namespace tps
