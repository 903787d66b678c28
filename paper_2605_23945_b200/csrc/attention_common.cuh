// Shared pieces of the paged decode-attention kernels (attention.cu, attention_balanced.cu).
#pragma once
#include "common.cuh"
#include "decode_ops.cuh"

namespace tps {

#ifndef ATTN_STAGES
#define ATTN_STAGES 3
#endif
constexpr int kPage = 64;          // tokens per KV page
constexpr int kAttnThreads = 128;  // 4 warps x 16 tokens of a page
constexpr int kAttnStages = ATTN_STAGES;  // cp.async ring depth (pages)
constexpr int kBalMaxRows = 512;   // rows per launch of the page-balanced schedule

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* smem) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(smem)));
}

// One 64-token page of one KV head through the tensor pipe: warp w owns tokens
// [16w, 16w+16) of the page. K and V tiles are [64][D] bf16 in smem with the
// 16-byte chunk index XOR-swizzled by (row & 7). Updates the warp's running
// (max, sum, O) state for the 16 query rows (the G heads of the KV group).
// Element offset of (token row t, 16-byte chunk cc) in a staged [64][D] page tile: the cp.async
// layout is row-major with the chunk index XOR-swizzled by (t & 7); the TMA layout (HALVES) is
// [D/64][64][64] as written by SWIZZLE_128B boxes of 64 columns -- the same XOR inside each
// 128-byte row, so fragment loads stay bank-conflict free in both.
template <int D, bool HALVES>
__device__ __forceinline__ int tile_off(int t, int cc) {
  if constexpr (HALVES) return (cc >> 3) * (kPage * 64) + t * 64 + (((cc & 7) ^ (t & 7)) * 8);
  else return t * D + ((cc ^ (t & 7)) * 8);
}

template <int D, bool HALVES = false>
__device__ __forceinline__ void attend_page(const __nv_bfloat16* K, const __nv_bfloat16* V,
                                            const uint32_t (&qa)[D / 16][4], int tok0, int ctx,
                                            float scale_log2, float (&m_r)[2], float (&l_r)[2],
                                            float (&o)[D / 8][4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  float s[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
    const int t = warp * 16 + nt * 8 + g;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(K + tile_off<D, HALVES>(t, 2 * ks) + 2 * c);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(K + tile_off<D, HALVES>(t, 2 * ks + 1) + 2 * c);
      mma16816(s[nt], qa[ks], b0, b1);
    }
  }
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int tok = tok0 + warp * 16 + nt * 8 + 2 * c + (e & 1);
      s[nt][e] = (tok < ctx) ? s[nt][e] * scale_log2 : -INFINITY;
    }
  float mx[2];
  mx[0] = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
  mx[1] = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
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
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = e >> 1;
      const float p = (mnew[r] == -INFINITY) ? 0.f : exp2f(s[nt][e] - mnew[r]);
      s[nt][e] = p;
      rs[r] += p;
    }
  l_r[0] = l_r[0] * alpha[0] + rs[0];
  l_r[1] = l_r[1] * alpha[1] + rs[1];
  // once the running max has settled the rescale is the identity: skip it
  if (!__all_sync(0xffffffffu, alpha[0] == 1.f && alpha[1] == 1.f)) {
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= alpha[0];
      o[i][1] *= alpha[0];
      o[i][2] *= alpha[1];
      o[i][3] *= alpha[1];
    }
  }
  uint32_t pa[4];
  pa[0] = pack_bf16(s[0][0], s[0][1]);
  pa[1] = pack_bf16(s[0][2], s[0][3]);
  pa[2] = pack_bf16(s[1][0], s[1][1]);
  pa[3] = pack_bf16(s[1][2], s[1][3]);
  const int vrow = warp * 16 + (lane & 15);
#pragma unroll
  for (int dn2 = 0; dn2 < D / 16; ++dn2) {
    const int chunk = 2 * dn2 + (lane >> 4);
    uint32_t r[4];
    ldmatrix_x4_trans(r, V + tile_off<D, HALVES>(vrow, chunk));
    mma16816(o[2 * dn2], pa, r[0], r[1]);
    mma16816(o[2 * dn2 + 1], pa, r[2], r[3]);
  }
}

// Q fragments (16 query rows = the G heads of a KV group, zero-padded) from global q.
template <int D>
__device__ __forceinline__ void load_q_frags(uint32_t (&qa)[D / 16][4], const __nv_bfloat16* q0, int G) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int d0 = ks * 16 + 2 * c;
    // q is written by the predecessor kernel, which may still have been running when this grid
    // started (PDL): coherent L2 loads, never the non-coherent read-only path
    qa[ks][0] = (g < G) ? __ldcg(reinterpret_cast<const unsigned int*>(q0 + g * D + d0)) : 0u;
    qa[ks][1] = (g + 8 < G) ? __ldcg(reinterpret_cast<const unsigned int*>(q0 + (g + 8) * D + d0)) : 0u;
    qa[ks][2] = (g < G) ? __ldcg(reinterpret_cast<const unsigned int*>(q0 + g * D + d0 + 8)) : 0u;
    qa[ks][3] = (g + 8 < G) ? __ldcg(reinterpret_cast<const unsigned int*>(q0 + (g + 8) * D + d0 + 8)) : 0u;
  }
}

}  // namespace tps
