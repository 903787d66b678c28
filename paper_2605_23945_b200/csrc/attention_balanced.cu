// Page-balanced persistent paged decode attention (sm_100a) -- the default attention.
//
// Same math as paged_attn_kernel (attention.cu) and the same cost model: the KV
// term of oracle_decode_latency, one pass over every live token's K/V head slice
// (tpshift/latency.py:123). What changes is the schedule. A decode batch is
// ragged (every sample sits at its own position), and a split count fixed at
// graph-capture time cannot follow it: one long sample serialises on its few
// CTAs while short ones finish early, and a grid that is not a whole number of
// resident waves leaves SMs idle in the last wave. Here the work is a flat list
// of units -- (row, kv head, page), 16 KB of K + 16 KB of V each (D = 128) --
// and the grid is exactly the resident CTA capacity (2 per SM): CTA c takes
// units [c*W/C, (c+1)*W/C). Every CTA streams the same number of bytes whatever
// the context lengths; its cp.async ring runs straight across segment (row,
// head) boundaries, and a segment cut between CTAs is finished by the last
// piece to arrive (log-sum-exp merge of at most a few partial states).
//
// Decode launches (row_pos == NULL) start streaming before the programmatic
// dependent launch wait: every cached token except the current one was written
// by earlier steps, so the first pages are issued while the QKV/RoPE kernel is
// still finishing; the current token's K/V row and q are read after the wait
// (the row is patched into a page that was issued early).
#include "attention_common.cuh"

namespace tps {

constexpr int kBalMinUnits = 2;   // pages per CTA floor
constexpr int kBalMaxCuts = 12;   // a segment spans <= ~kBalMaxCuts + 2 CTAs (merge length)
constexpr int kBalScratch = 4 * 16 * 32;  // floats: cross-warp merge (32 columns per round) / merge factors
constexpr int kBalTab = 256;      // unit table ring (page offsets), refilled 128 units at a time

template <int D>
static constexpr int bal_smem() {
  return 2 * kAttnStages * kPage * D * 2      // K and V rings
         + kBalScratch * 4                    // merge scratch
         + 2 * 4 * 16 * 4                     // per-warp (max, sum)
         + 2 * (kBalMaxRows + 1) * 4          // per-row ctx and unit prefix
         + kBalTab * 4;                       // unit table
}

template <int D, bool TMA>
__global__ void __launch_bounds__(kAttnThreads) paged_attn_balanced_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __nv_bfloat16* __restrict__ v_cache, const int* __restrict__ row_slot,
    const int* __restrict__ pos_by_slot, const int* __restrict__ row_pos, const int* __restrict__ page_table,
    int max_pages, int B, int nq, int nkv, int G, float scale_log2, float* __restrict__ part_m,
    float* __restrict__ part_l, float* __restrict__ part_o, unsigned int* __restrict__ merge_ctr,
    __nv_bfloat16* __restrict__ out, const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv) {
  constexpr int CPR = D / 8;
  constexpr int TILE = kPage * D;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem_base = TMA ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023))
                           : smem_raw;  // (SWIZZLE_128B boxes land on 1024-byte boundaries)
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem_base);
  __nv_bfloat16* sv = sk + kAttnStages * TILE;
  float* scr = reinterpret_cast<float*>(sv + kAttnStages * TILE);  // [4 warps][16][32]
  float* wm = scr + kBalScratch;                                    // [4][16]
  float* wl = wm + 64;                                              // [4][16]
  int* sctx = reinterpret_cast<int*>(wl + 64);                      // [B] context length
  int* pre = sctx + kBalMaxRows + 1;                                // [B+1] units before row b
  int* utab = pre + kBalMaxRows + 1;                                // [kBalTab] page * nkv + head
  __shared__ int s_wsum[4], s_wmax[4];
  __shared__ int s_last, s_cf, s_cl;
  __shared__ __align__(8) uint64_t full_bar[kAttnStages];
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < kAttnStages; ++i) mbar_init(&full_bar[i], 1);
      fence_barrier_init();
    }
    __syncthreads();
  }

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, c4 = lane & 3;
  const bool decode = row_pos == nullptr;
  pdl_launch_dependents();  // the O projection may launch and prefetch its weights now
  const unsigned int trs = trace_begin(kTrAttnBal);
  if (!decode) pdl_wait();  // prefill: earlier rows of this chunk were appended by the previous kernel

  // ---- unit prefix over rows: row b owns nkv * ceil(ctx_b / 64) units ----
  const int per = (B + kAttnThreads - 1) / kAttnThreads;
  const int r0 = tid * per, r1 = min(B, r0 + per);
  int loc = 0, locmax = 0;
  for (int r = r0; r < r1; ++r) {
    const int slot = row_slot[r];
    const int ctx = slot >= 0 ? (decode ? pos_by_slot[slot] : row_pos[r]) + 1 : 0;
    sctx[r] = ctx;
    const int np = (ctx + kPage - 1) / kPage;
    loc += np;
    locmax = max(locmax, np);
  }
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int wmx = __reduce_max_sync(0xffffffffu, locmax);
  if (lane == 31) s_wsum[warp] = incl;
  if (lane == 0) s_wmax[warp] = wmx;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += s_wsum[w];
  {
    int run = base + incl - loc;
    for (int r = r0; r < r1; ++r) {
      pre[r] = run * nkv;
      run += (sctx[r] + kPage - 1) / kPage;
    }
  }
  if (tid == 0) pre[B] = (s_wsum[0] + s_wsum[1] + s_wsum[2] + s_wsum[3]) * nkv;
  __syncthreads();
  const long long W = pre[B];
  const int nb_max = max(max(s_wmax[0], s_wmax[1]), max(s_wmax[2], s_wmax[3]));

  // ---- this CTA's unit range: C equal slices of the W units ----
  long long ceff = W / kBalMinUnits;
  if (ceff > gridDim.x) ceff = gridDim.x;
  if (nb_max > 0 && ceff > (long long)kBalMaxCuts * W / nb_max) ceff = (long long)kBalMaxCuts * W / nb_max;
  if (ceff < 1) ceff = 1;
  const int C = (int)ceff;
  auto start_of = [&](int c) -> long long { return (long long)c * W / C; };
  auto cta_of = [&](long long u) -> int {
    int c = (int)(u * C / W);
    while (c + 1 < C && start_of(c + 1) <= u) ++c;
    while (c > 0 && start_of(c) > u) --c;
    return c;
  };
  auto row_of = [&](long long u) -> int {  // pre[b] <= u < pre[b + 1]
    int lo = 0, hi = B;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= u) lo = mid; else hi = mid;
    }
    return lo;
  };
  const int cta = blockIdx.x;
  const long long u0 = cta < C ? start_of(cta) : 0, u1 = cta < C ? start_of(cta + 1) : 0;
  const int n_units = (int)(u1 - u0);

  // unit table: global page-slice index of units [j0, j0 + 128), one thread per unit
  auto fill = [&](int j0) {
    const int j = j0 + tid;
    if (j < n_units) {
      const long long u = u0 + j;
      const int b = row_of(u);
      const int nb = (pre[b + 1] - pre[b]) / nkv;
      const int off = (int)(u - pre[b]);
      const int h = off / nb, p = off - h * nb;
      utab[j & (kBalTab - 1)] = page_table[(size_t)row_slot[b] * max_pages + p] * nkv + h;
    }
  };
  auto load_unit = [&](int j, int st) {
    if constexpr (TMA) {
      if (tid == 0) {
        const int row0 = utab[j & (kBalTab - 1)] * kPage;
        const uint64_t pol = policy_evict_first();
        mbar_arrive_expect_tx(&full_bar[st], 2 * TILE * 2);
#pragma unroll
        for (int hh = 0; hh < D / 64; ++hh) {
          tma_load_2d(sk + st * TILE + hh * kPage * 64, &tmk, &full_bar[st], hh * 64, row0, pol);
          tma_load_2d(sv + st * TILE + hh * kPage * 64, &tmv, &full_bar[st], hh * 64, row0, pol);
        }
      }
      return;
    }
    const size_t goff = (size_t)utab[j & (kBalTab - 1)] * TILE;
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
  };

  fill(0);
  fill(128);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kAttnStages - 1; ++i) {
    if (i < n_units) load_unit(i, i);
    cp_async_commit();
  }
  if (decode) pdl_wait();
  trace_mark(trs, 2);

  // padding rows (slot < 0) have no units: CTA 0 zeroes their output
  if (cta == 0) {
    for (int r = 0; r < B; ++r)
      if (sctx[r] == 0)
        for (int i = tid; i < nq * D; i += kAttnThreads) out[(size_t)r * nq * D + i] = __float2bfloat16(0.f);
  }

  // consumer cursor over (row b, kv head h, page p); nb = pages of row b
  int b = 0, h = 0, p = 0, nb = 1;
  if (n_units > 0) {
    b = row_of(u0);
    nb = (pre[b + 1] - pre[b]) / nkv;
    const int off = (int)(u0 - pre[b]);
    h = off / nb;
    p = off - h * nb;
  }
  uint32_t qa[D / 16][4];
  float m_r[2], l_r[2];
  float o[D / 8][4];
  int piece_first = 0;  // first iteration of the current piece
  for (int it = 0; it < n_units; ++it) {
    if constexpr (TMA) {
      __syncthreads();  // every warp is done with the stage the next load overwrites
      const int nxt = it + kAttnStages - 1;
      if ((nxt & 127) == 0 && nxt >= 128) {
        fill(nxt + 128);  // slots of units [nxt-128, nxt) are free
        __syncthreads();
      }
      if (nxt < n_units) {
        if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        load_unit(nxt, nxt % kAttnStages);
      }
      mbar_wait(&full_bar[it % kAttnStages], (uint32_t)((it / kAttnStages) & 1));
    } else {
      cp_async_wait<kAttnStages - 2>();
      __syncthreads();
      const int nxt = it + kAttnStages - 1;
      if ((nxt & 127) == 0 && nxt >= 128) fill(nxt + 128);  // slots of units [nxt-128, nxt) are free
      if (nxt < n_units) load_unit(nxt, nxt % kAttnStages);
      cp_async_commit();
    }
    const int ctx = sctx[b];
    const int st = it % kAttnStages;
    if (it == 0 || p == 0) {
      piece_first = it;
      load_q_frags<D>(qa, q + ((size_t)b * nq + h * G) * D, G);
      m_r[0] = m_r[1] = -INFINITY;
      l_r[0] = l_r[1] = 0.f;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    }
    if (decode && it < kAttnStages - 1 && p == nb - 1) {
      // issued before the PDL wait: refresh the current token's K/V row
      const int r = (ctx - 1) % kPage;
      const size_t goff = (size_t)utab[it] * TILE + (size_t)r * D;
      for (int i = tid; i < 2 * CPR; i += kAttnThreads) {
        const bool is_v = i >= CPR;
        const int cc = i % CPR;
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>((is_v ? v_cache : k_cache) + goff) + cc);
        *reinterpret_cast<uint4*>((is_v ? sv : sk) + st * TILE + tile_off<D, TMA>(r, cc)) = v;
      }
      __syncthreads();
    }
    attend_page<D, TMA>(sk + st * TILE, sv + st * TILE, qa, p * kPage, ctx, scale_log2, m_r, l_r, o);

    const bool seg_end = p == nb - 1;
    if (seg_end || it == n_units - 1) {
      // ---- piece end: combine the 4 warps, then output or partial + merge ----
      const int p_first = p - (it - piece_first);
      const bool full = (p_first == 0 && seg_end);
      const int slotp = piece_first == 0 ? 0 : 1;
      const int head0 = h * G;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
      }
      if (c4 == 0) {
        wm[warp * 16 + g] = m_r[0];
        wm[warp * 16 + g + 8] = m_r[1];
        wl[warp * 16 + g] = l_r[0];
        wl[warp * 16 + g + 8] = l_r[1];
      }
      const size_t pidx = ((size_t)cta * 2 + slotp) * 16;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int d = j * 8 + 2 * c4;
          scr[(warp * 16 + g) * 32 + d] = o[cc * 4 + j][0];
          scr[(warp * 16 + g) * 32 + d + 1] = o[cc * 4 + j][1];
          scr[(warp * 16 + g + 8) * 32 + d] = o[cc * 4 + j][2];
          scr[(warp * 16 + g + 8) * 32 + d + 1] = o[cc * 4 + j][3];
        }
        __syncthreads();
        for (int i = tid; i < G * 32; i += kAttnThreads) {
          const int hh = i >> 5, d = i & 31;
          float M = -INFINITY;
#pragma unroll
          for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * 16 + hh]);
          float L = 0.f, acc = 0.f;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const float mw = wm[w * 16 + hh];
            const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
            L += wl[w * 16 + hh] * f;
            acc += scr[(w * 16 + hh) * 32 + d] * f;
          }
          if (full) {
            out[((size_t)b * nq + head0 + hh) * D + cc * 32 + d] = f2bf(L > 0.f ? acc / L : 0.f);
          } else {
            part_o[(pidx + hh) * D + cc * 32 + d] = acc;
            if (cc == 0 && d == 0) {
              part_m[pidx + hh] = M;
              part_l[pidx + hh] = L;
            }
          }
        }
        __syncthreads();
      }
      if (!full) {
        // segment cut between CTAs: the last piece to arrive merges
        const long long s0 = pre[b] + (long long)h * nb;
        __threadfence();
        __syncthreads();
        if (tid == 0) {
          const int cf = cta_of(s0), cl = cta_of(s0 + nb - 1);
          const unsigned int prev = atomicAdd(&merge_ctr[b * nkv + h], 1u);
          s_last = (prev == (unsigned int)(cl - cf));
          s_cf = cf;
          s_cl = cl;
        }
        __syncthreads();
        if (s_last) {
          __threadfence();
          const int cf = s_cf, np = s_cl - s_cf + 1;
          // piece slot of CTA c in this segment: 0 if the segment is its first piece
          auto pslot = [&](int c) -> size_t { return ((size_t)c * 2 + (start_of(c) >= s0 ? 0 : 1)) * 16; };
          float* fac = scr;  // [G][np] rescale factors; 1/L per head in wm
          for (int hh = warp; hh < G; hh += 4) {
            float M = -INFINITY;
            for (int j = lane; j < np; j += 32) M = fmaxf(M, __ldcg(part_m + pslot(cf + j) + hh));
            M = warp_max(M);
            float L = 0.f;
            for (int j = lane; j < np; j += 32) {
              const size_t pi = pslot(cf + j) + hh;
              const float ms = __ldcg(part_m + pi);
              const float f = (ms == -INFINITY || M == -INFINITY) ? 0.f : exp2f(ms - M);
              fac[hh * np + j] = f;
              L += __ldcg(part_l + pi) * f;
            }
            L = warp_sum(L);
            if (lane == 0) wm[hh] = L > 0.f ? 1.f / L : 0.f;
          }
          __syncthreads();
          // O: each thread owns up to NC float4 columns of the G x D output; 4 pieces per batch
          constexpr int D4 = D / 4;
          constexpr int NC = (16 * D4 + kAttnThreads - 1) / kAttnThreads;
          const int ncol = G * D4;
          float4 acc[NC];
#pragma unroll
          for (int k = 0; k < NC; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int j0 = 0; j0 < np; j0 += 4) {
            float4 v[4][NC];
            size_t ps[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) ps[jj] = j0 + jj < np ? pslot(cf + j0 + jj) : 0;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int k = 0; k < NC; ++k) {
                const int col = tid + k * kAttnThreads;
                v[jj][k] = (col < ncol && j0 + jj < np)
                               ? __ldcg(reinterpret_cast<const float4*>(part_o + (ps[jj] + col / D4) * D) + col % D4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int k = 0; k < NC; ++k) {
                const int col = tid + k * kAttnThreads;
                const float f = (col < ncol && j0 + jj < np) ? fac[(col / D4) * np + j0 + jj] : 0.f;
                acc[k].x += v[jj][k].x * f;
                acc[k].y += v[jj][k].y * f;
                acc[k].z += v[jj][k].z * f;
                acc[k].w += v[jj][k].w * f;
              }
          }
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            const int col = tid + k * kAttnThreads;
            if (col < ncol) {
              const int hh = col / D4, d = (col % D4) * 4;
              const float s = wm[hh];
              uint2 pk;
              pk.x = pack_bf16(acc[k].x * s, acc[k].y * s);
              pk.y = pack_bf16(acc[k].z * s, acc[k].w * s);
              *reinterpret_cast<uint2*>(out + ((size_t)b * nq + head0 + hh) * D + d) = pk;
            }
          }
          if (tid == 0) merge_ctr[b * nkv + h] = 0u;  // re-arm for the next launch / graph replay
          __syncthreads();
        }
      }
    }
    // advance the cursor
    if (++p == nb) {
      p = 0;
      if (++h == nkv) {
        h = 0;
        if (it + 1 < n_units) {
          do ++b; while (pre[b + 1] == pre[b]);
          nb = (pre[b + 1] - pre[b]) / nkv;
        }
      }
    }
  }
  cp_async_wait<0>();
  trace_mark(trs, 3);
}

static int g_bal_grid[2] = {0, 0};  // resident CTA capacity for D = 64, 128

// TPS_ATTN_TMA_BAL=0: the page-balanced form stages its pages with cp.async instead of TMA boxes
static int g_bal_tma = [] {
  const char* e = getenv("TPS_ATTN_TMA_BAL");
  return e ? atoi(e) : 1;
}();

int make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

int configure_attention_balanced() {
  int dev = 0, sms = 0;
  TPS_CUDA_TRY(cudaGetDevice(&dev));
  TPS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_balanced_kernel<128, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, bal_smem<128>()));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_balanced_kernel<128, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, bal_smem<128>() + 1024));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_attn_balanced_kernel<64, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, bal_smem<64>()));
  TPS_MAX_CARVEOUT((paged_attn_balanced_kernel<128, false>));
  TPS_MAX_CARVEOUT((paged_attn_balanced_kernel<128, true>));
  TPS_MAX_CARVEOUT((paged_attn_balanced_kernel<64, false>));
  int occ = 0;
  TPS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, paged_attn_balanced_kernel<64, false>,
                                                             kAttnThreads, bal_smem<64>()));
  g_bal_grid[0] = occ * sms;
  int occ_t = 0;
  TPS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, paged_attn_balanced_kernel<128, false>,
                                                             kAttnThreads, bal_smem<128>()));
  TPS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, paged_attn_balanced_kernel<128, true>,
                                                             kAttnThreads, bal_smem<128>() + 1024));
  if (occ_t < occ) g_bal_tma = 0;  // (the TMA form only where it keeps the residency)
  g_bal_grid[1] = occ * sms;
  if (g_bal_grid[0] <= 0 || g_bal_grid[1] <= 0) return fail(kCuda, "balanced attention: zero occupancy");
  return kOk;
}

// Grid of the balanced kernel (fixed per head dim: graph-capture safe). Before
// tps_init the B200 figure (2 CTAs x 148 SMs for D = 128) is assumed.
int attn_balanced_grid(int D) {
  const int i = D == 64 ? 0 : 1;
  if (g_bal_grid[i] > 0) return g_bal_grid[i];
  return (D == 64 ? 4 : 2) * kNumSMs;
}

int paged_attention_balanced(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                             const int* pos_by_slot, const int* row_pos, const int* page_table, int max_pages,
                             int B, int nq, int nkv, int D, float* part_m, float* part_l, float* part_o,
                             unsigned int* merge_ctr, void* out, cudaStream_t st) {
  TPS_CHECK_ARG(B <= kBalMaxRows, "paged_attention: the balanced schedule takes at most 512 rows per launch");
  const int G = nq / nkv;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  const auto* qq = reinterpret_cast<const __nv_bfloat16*>(q);
  const auto* kk = reinterpret_cast<const __nv_bfloat16*>(k_cache);
  const auto* vv = reinterpret_cast<const __nv_bfloat16*>(v_cache);
  auto* oo = reinterpret_cast<__nv_bfloat16*>(out);
  const dim3 grid(attn_balanced_grid(D));
  CUtensorMap tmk{}, tmv{};
  if (D == 128 && g_bal_tma) {
    int rc = make_tmap_bf16(&tmk, k_cache, 1LL << 28, D, D, kPage);
    if (!rc) rc = make_tmap_bf16(&tmv, v_cache, 1LL << 28, D, D, kPage);
    if (rc) return rc;
    return launch_k(paged_attn_balanced_kernel<128, true>, grid, dim3(kAttnThreads), bal_smem<128>() + 1024, st, true,
                    qq, kk, vv, row_slot, pos_by_slot, row_pos, page_table, max_pages, B, nq, nkv, G, scale_log2,
                    part_m, part_l, part_o, merge_ctr, oo, tmk, tmv);
  }
  if (D == 128)
    return launch_k(paged_attn_balanced_kernel<128, false>, grid, dim3(kAttnThreads), bal_smem<128>(), st, true, qq,
                    kk, vv, row_slot, pos_by_slot, row_pos, page_table, max_pages, B, nq, nkv, G, scale_log2, part_m,
                    part_l, part_o, merge_ctr, oo, tmk, tmv);
  if (D == 64)
    return launch_k(paged_attn_balanced_kernel<64, false>, grid, dim3(kAttnThreads), bal_smem<64>(), st, true, qq, kk,
                    vv, row_slot, pos_by_slot, row_pos, page_table, max_pages, B, nq, nkv, G, scale_log2, part_m,
                    part_l, part_o, merge_ctr, oo, tmk, tmv);
  return fail(kInvalid, "paged_attention: head_dim must be 64 or 128");
}

int trace_register_attention_bal(uint64_t* p, unsigned int* c, unsigned int n) {
  return trace_register(p, c, n);
}

}  // namespace tps
