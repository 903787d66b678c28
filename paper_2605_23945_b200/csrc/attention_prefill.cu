// Chunked-prefill attention over the paged KV cache (sm_100a).
//
// A prefill chunk holds many (sample, position) rows of the same samples (position-major:
// row i of a 512-row chunk of 64 prompts is sample i % 64 at one of 8 consecutive
// positions). The decode kernels treat every row as its own segment, so each sample's
// pages are re-read once per row and per KV head. Here the rows of one sample are a
// *group* (host-built table, up to 16 positions and at most 64 query rows per KV head):
// one CTA per (group, KV head) streams the sample's pages once, and each of its 4 warps
// owns one 16-row MMA tile of (position, query head) rows over every token of the page,
// with a per-row causal limit (token <= the row's position). The result per row is the
// same attention the decode kernels compute (softmax over tokens 0..pos of its sample);
// this is the prefill / recompute term of the reference's cost model
// (tpshift/latency.py:136-152, tpshift/switchcost.py:203-219).
#include "attention_common.cuh"

namespace tps {

constexpr int kPfMaxPos = 16;   // positions per group
constexpr int kPfMaxRows = 64;  // (position, head) rows per group = 4 warps x 16

// One 64-token page for a warp's 16 query rows (all 64 tokens: 8 score n-tiles, 4 PV k-steps).
// lim[r]: row r's token limit (tokens < lim attend), r = 0 for row g, 1 for row g + 8.
template <int D>
__device__ __forceinline__ void attend_page_rows(const __nv_bfloat16* K, const __nv_bfloat16* V,
                                                 const uint32_t (&qa)[D / 16][4], int tok0, const int (&lim)[2],
                                                 float scale_log2, float (&m_r)[2], float (&l_r)[2],
                                                 float (&o)[D / 8][4]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  float s[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
    const int t = nt * 8 + g;
    const __nv_bfloat16* krow = K + t * D + 2 * c;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(krow + (((2 * ks) ^ (t & 7)) * 8));
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(krow + (((2 * ks + 1) ^ (t & 7)) * 8));
      mma16816(s[nt], qa[ks], b0, b1);
    }
  }
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int tok = tok0 + nt * 8 + 2 * c + (e & 1);
      s[nt][e] = (tok < lim[e >> 1]) ? s[nt][e] * scale_log2 : -INFINITY;
    }
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    mx[0] = fmaxf(mx[0], fmaxf(s[nt][0], s[nt][1]));
    mx[1] = fmaxf(mx[1], fmaxf(s[nt][2], s[nt][3]));
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
  }
  float alpha[2], mnew[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    mnew[r] = fmaxf(m_r[r], mx[r]);
    alpha[r] = (mnew[r] == -INFINITY) ? 1.f : exp2f(m_r[r] - mnew[r]);
    m_r[r] = mnew[r];
  }
  float rs[2] = {0.f, 0.f};
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = e >> 1;
      const float p = (mnew[r] == -INFINITY) ? 0.f : exp2f(s[nt][e] - mnew[r]);
      s[nt][e] = p;
      rs[r] += p;
    }
  l_r[0] = l_r[0] * alpha[0] + rs[0];
  l_r[1] = l_r[1] * alpha[1] + rs[1];
  if (!__all_sync(0xffffffffu, alpha[0] == 1.f && alpha[1] == 1.f)) {
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= alpha[0];
      o[i][1] *= alpha[0];
      o[i][2] *= alpha[1];
      o[i][3] *= alpha[1];
    }
  }
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) {  // 16 tokens per PV k-step
    uint32_t pa[4];
    pa[0] = pack_bf16(s[2 * kt][0], s[2 * kt][1]);
    pa[1] = pack_bf16(s[2 * kt][2], s[2 * kt][3]);
    pa[2] = pack_bf16(s[2 * kt + 1][0], s[2 * kt + 1][1]);
    pa[3] = pack_bf16(s[2 * kt + 1][2], s[2 * kt + 1][3]);
    const int vrow = kt * 16 + (lane & 15);
#pragma unroll
    for (int dn2 = 0; dn2 < D / 16; ++dn2) {
      const int chunk = 2 * dn2 + (lane >> 4);
      uint32_t r[4];
      ldmatrix_x4_trans(r, V + vrow * D + ((chunk ^ (vrow & 7)) * 8));
      mma16816(o[2 * dn2], pa, r[0], r[1]);
      mma16816(o[2 * dn2 + 1], pa, r[2], r[3]);
    }
  }
}

// grid = (kv head, group stride); group y: grp_n[y] rows grp_rows[y][0..n) of one sample.
template <int D>
__global__ void __launch_bounds__(kAttnThreads) paged_prefill_attn_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_cache,
    const __nv_bfloat16* __restrict__ v_cache, const int* __restrict__ row_slot, const int* __restrict__ row_pos,
    const int* __restrict__ grp_rows, const int* __restrict__ grp_n, const int* __restrict__ page_table,
    int max_pages, int max_groups, int nq, int nkv, int G, float scale_log2, __nv_bfloat16* __restrict__ out) {
  constexpr int CPR = D / 8;
  constexpr int TILE = kPage * D;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sv = sk + kAttnStages * TILE;
  __shared__ int s_row[kPfMaxPos], s_lim[kPfMaxPos];

  const int kvh = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, c = lane & 3;
  pdl_launch_dependents();
  const unsigned int trs = trace_begin(kTrAttnPrefill);
  pdl_wait();  // this chunk's K/V rows were appended by the previous kernel
  trace_mark(trs, 2);
  // groups strided over a grid of at most one resident wave
  for (int grp = blockIdx.y; grp < max_groups; grp += gridDim.y) {
    const int n = grp_n[grp];
    if (n <= 0) break;  // groups are numbered densely from 0
    if (tid < n) {
      const int r = grp_rows[grp * kPfMaxPos + tid];
      s_row[tid] = r;
      s_lim[tid] = row_pos[r] + 1;
    }
    __syncthreads();
    const int slot = row_slot[s_row[0]];
    int ctx = 0;
    for (int i = 0; i < n; ++i) ctx = max(ctx, s_lim[i]);
    const int npages = (ctx + kPage - 1) / kPage;
    const int head0 = kvh * G;
    const int* pt = page_table + (size_t)slot * max_pages;

    // this warp's 16 rows: m = warp * 16 + {g, g + 8} -> (position index m / G, head m % G)
    int lim[2], orow[2], ohead[2];
    uint32_t qa[D / 16][4];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int m = warp * 16 + g + 8 * r;
      const int pi = m / G;
      const bool ok = pi < n;
      orow[r] = ok ? s_row[pi] : -1;
      ohead[r] = m % G;
      lim[r] = ok ? s_lim[pi] : 0;
    }
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const int d0 = ks * 16 + 2 * c;
      const __nv_bfloat16* q0 = orow[0] >= 0 ? q + ((size_t)orow[0] * nq + head0 + ohead[0]) * D : nullptr;
      const __nv_bfloat16* q1 = orow[1] >= 0 ? q + ((size_t)orow[1] * nq + head0 + ohead[1]) * D : nullptr;
      qa[ks][0] = q0 ? *reinterpret_cast<const uint32_t*>(q0 + d0) : 0u;
      qa[ks][1] = q1 ? *reinterpret_cast<const uint32_t*>(q1 + d0) : 0u;
      qa[ks][2] = q0 ? *reinterpret_cast<const uint32_t*>(q0 + d0 + 8) : 0u;
      qa[ks][3] = q1 ? *reinterpret_cast<const uint32_t*>(q1 + d0 + 8) : 0u;
    }

    auto load_page = [&](int p, int st) {
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
    };
#pragma unroll
    for (int i = 0; i < kAttnStages - 1; ++i) {
      if (i < npages) load_page(i, i);
      cp_async_commit();
    }
    float m_r[2] = {-INFINITY, -INFINITY};
    float l_r[2] = {0.f, 0.f};
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    const bool active = warp * 16 < n * G;  // warps past the group's rows only help stream
    for (int it = 0; it < npages; ++it) {
      cp_async_wait<kAttnStages - 2>();
      __syncthreads();
      {
        const int nxt = it + kAttnStages - 1;
        if (nxt < npages) load_page(nxt, nxt % kAttnStages);
        cp_async_commit();
      }
      const int st = it % kAttnStages;
      if (active)
        attend_page_rows<D>(sk + st * TILE, sv + st * TILE, qa, it * kPage, lim, scale_log2, m_r, l_r, o);
    }
    cp_async_wait<0>();
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
      l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (orow[r] < 0) continue;
      const float inv = l_r[r] > 0.f ? 1.f / l_r[r] : 0.f;
      __nv_bfloat16* dst = out + ((size_t)orow[r] * nq + head0 + ohead[r]) * D;
#pragma unroll
      for (int dn = 0; dn < D / 8; ++dn) {
        const int d = dn * 8 + 2 * c;
        *reinterpret_cast<__nv_bfloat162*>(dst + d) = __floats2bfloat162_rn(o[dn][2 * r] * inv, o[dn][2 * r + 1] * inv);
      }
    }
    __syncthreads();  // s_row / s_lim and the ring are reused by the next group
  }
  trace_mark(trs, 3);
}

template <int D>
static constexpr int pf_smem() {
  return 2 * kAttnStages * kPage * D * 2;
}

int configure_attention_prefill() {
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_prefill_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    pf_smem<128>()));
  TPS_CUDA_TRY(cudaFuncSetAttribute(paged_prefill_attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    pf_smem<64>()));
  TPS_MAX_CARVEOUT(paged_prefill_attn_kernel<128>);
  TPS_MAX_CARVEOUT(paged_prefill_attn_kernel<64>);
  return kOk;
}

int prefill_group_positions(int G) {
  if (G < 1 || G > kPfMaxRows) return 0;
  const int p = kPfMaxRows / G;
  return p < kPfMaxPos ? p : kPfMaxPos;
}

int paged_prefill_attention(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                            const int* row_pos, const int* grp_rows, const int* grp_n, int max_groups,
                            const int* page_table, int max_pages, int nq, int nkv, int D, void* out,
                            cudaStream_t st) {
  TPS_CHECK_ARG(nkv > 0 && nq % nkv == 0 && max_groups > 0, "prefill_attention: bad shape");
  const int G = nq / nkv;
  TPS_CHECK_ARG(G <= kPfMaxRows, "prefill_attention: at most 64 query heads per KV head");
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  // one resident wave (2 CTAs per SM), each CTA striding over groups
  int gy = (2 * kNumSMs + nkv - 1) / nkv;
  if (gy > max_groups) gy = max_groups;
  const dim3 grid(nkv, gy);
  const auto* qq = reinterpret_cast<const __nv_bfloat16*>(q);
  const auto* kk = reinterpret_cast<const __nv_bfloat16*>(k_cache);
  const auto* vv = reinterpret_cast<const __nv_bfloat16*>(v_cache);
  auto* oo = reinterpret_cast<__nv_bfloat16*>(out);
  if (D == 128)
    return launch_k(paged_prefill_attn_kernel<128>, grid, dim3(kAttnThreads), pf_smem<128>(), st, true, qq, kk, vv,
                    row_slot, row_pos, grp_rows, grp_n, page_table, max_pages, max_groups, nq, nkv, G, scale_log2, oo);
  if (D == 64)
    return launch_k(paged_prefill_attn_kernel<64>, grid, dim3(kAttnThreads), pf_smem<64>(), st, true, qq, kk, vv,
                    row_slot, row_pos, grp_rows, grp_n, page_table, max_pages, max_groups, nq, nkv, G, scale_log2, oo);
  return fail(kInvalid, "prefill_attention: head_dim must be 64 or 128");
}

int trace_register_attention_prefill(uint64_t* p, unsigned int* c, unsigned int n) { return trace_register(p, c, n); }

}  // namespace tps
