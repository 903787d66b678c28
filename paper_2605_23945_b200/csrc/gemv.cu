// Warp-shuffle GEMV for tail decode batches (b <= 4): the `north_star` "warp-shuffle
// vectorised GEMV at tail batch sizes" (VERDICT row N1). Same output contracts as the
// tcgen05 projection family it stands in for at the tail (gemm_tcgen05.cu), so the executor
// swaps one call for the other:
//
//   tps_gemv          == tps_linear with splits = 1          (fp32 [b][n])
//   tps_gemv_silu     == tps_linear_silu                      (bf16 SwiGLU activations)
//   tps_gemv_push_ll  == tps_linear_push_ll_cluster           (one LL {value, tag} per element
//                                                              to every TP peer: fused allreduce push)
//   tps_gemv_argmax   == tps_linear_argmax                    (logits + a greedy candidate per
//                                                              (row, 128-column tile))
//
// Replaces the weight-traffic term of oracle_decode_latency (tpshift/latency.py:123-124) where
// the tensor-core tile's fixed costs (TMEM allocation, barrier ring, 128-row tiles with split-K
// partials round-tripping HBM) dominate a small TP shard.
//
// Layout: 256 threads = 8 warps, split into `groups` row groups of group_warps = 8 / groups
// warps. A row group owns kGvRows weight rows (one output each; SwiGLU: 2 outputs x {gate, up}
// rows of the interleaved 64-row blocks) and strides their K with 16-B vectors, two vectors per
// row in flight per thread (L1::no_allocate streaming loads; the activations, b x K bf16, are
// re-read through L1). Partial dot products are reduced with xor warp shuffles, then across the
// group's warps in a fixed order through shared memory, so every output is deterministic.
// Before the programmatic-dependent-launch wait each group asks the TMA engine to pull its
// first rows into L2 (cp.async.bulk.prefetch.L2): weights are never written by a decode step.
// Bound: HBM (weights); b <= 4 keeps the FMA work (8 b FMA per 16 B) under the CUDA-core rate.
#include <climits>

#include "common.cuh"
#include "decode_ops.cuh"

namespace tps {
namespace {

constexpr int kGvThreads = 256;
constexpr int kGvWarps = kGvThreads / 32;
constexpr int kGvRows = 4;   // weight rows per row group
constexpr int kGvMaxB = 4;   // batch rows per launch
constexpr int kGvTargetCtas = 2 * kNumSMs;

enum : int { kGvPartial = 0, kGvSilu = 1, kGvLL = 2, kGvArgmax = 3 };

struct GvArgs {
  const __nv_bfloat16* w;
  long long ldw;
  int n_out;  // outputs (SwiGLU: n / 2)
  int k;
  const __nv_bfloat16* x;
  long long ldx;
  int b;
  float* out;  // kGvPartial / kGvArgmax: fp32 [b][n_out]
  __nv_bfloat16* act;  // kGvSilu: bf16 [b][ld_act]
  long long ld_act;
  const uint64_t* epoch;  // kGvLL: tag = (*epoch) * tag_mult + tag_add
  uint32_t tag_mult, tag_add;
  ArgmaxCand* cand;  // kGvArgmax: [b][ntiles]
  int ntiles;
  int vocab0;
  int group_warps;  // 1, 2, 4 or 8
};

__device__ __forceinline__ uint4 ld_stream16(const __nv_bfloat16* p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p));
  return v;
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// 8 bf16 (little-endian pairs: element 2j in the low half) -> fp32 (exact)
__device__ __forceinline__ void bf16x8_f32(const uint4 v, float f[8]) {
  f[0] = __uint_as_float(v.x << 16);
  f[1] = __uint_as_float(v.x & 0xffff0000u);
  f[2] = __uint_as_float(v.y << 16);
  f[3] = __uint_as_float(v.y & 0xffff0000u);
  f[4] = __uint_as_float(v.z << 16);
  f[5] = __uint_as_float(v.z & 0xffff0000u);
  f[6] = __uint_as_float(v.w << 16);
  f[7] = __uint_as_float(v.w & 0xffff0000u);
}

// acc[r][i] += W[r][vec v] . X[i][vec v]
template <int NB>
__device__ __forceinline__ void gv_fma(float (&acc)[kGvRows][NB], const uint4 (&wv)[kGvRows], const GvArgs& a,
                                       int v) {
  float xf[NB][8];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int xi = i < a.b ? i : a.b - 1;  // rows >= b: any valid row, results discarded
    const uint4 xv = __ldg(reinterpret_cast<const uint4*>(a.x + (size_t)xi * a.ldx) + v);
    bf16x8_f32(xv, xf[i]);
  }
#pragma unroll
  for (int r = 0; r < kGvRows; ++r) {
    float wf[8];
    bf16x8_f32(wv[r], wf);
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[r][i] = fmaf(wf[e], xf[i][e], acc[r][i]);
  }
}

// output column of the group's weight row r (o0 = the group's first output)
template <int EPI>
__device__ __forceinline__ int gv_out_of(int o0, int r) {
  return EPI == kGvSilu ? o0 + (r >> 1) : o0 + r;
}
// weight row of output o, row r of the group (SwiGLU: blocks of 64 [gate | up] rows)
template <int EPI>
__device__ __forceinline__ int gv_row_of(int o, int r) {
  return EPI == kGvSilu ? (o >> 6) * 128 + (o & 63) + (r & 1) * 64 : o;
}

template <int NB, int EPI>
__global__ void __launch_bounds__(kGvThreads, 2) gemv_kernel(const __grid_constant__ GvArgs a,
                                                             const __grid_constant__ DstList dst) {
  __shared__ float red[kGvWarps][kGvRows * NB];
  __shared__ ArgmaxCand cs[kGvWarps][kGvRows * NB];
  const unsigned int trs = trace_begin(kTrGemv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = a.group_warps;
  const int groups = kGvWarps / gw;
  const int grp = warp / gw;
  const int gt = (warp - grp * gw) * 32 + lane;  // thread index inside the row group
  const int tk = gw * 32;
  const int nvec = a.k >> 3;
  constexpr int kOpg = EPI == kGvSilu ? kGvRows / 2 : kGvRows;  // outputs per group per pass
  const int sub_cols = kOpg * groups;
  const int cta_cols = EPI == kGvArgmax ? 128 : sub_cols;
  const int passes = cta_cols / sub_cols;
  const int col_base = blockIdx.x * cta_cols;

  // the first pass's weight rows into L2 while the producer of x finishes
  if (gt < kGvRows) {
    const int o = gv_out_of<EPI>(col_base + grp * kOpg, gt);
    if (o < a.n_out) prefetch_l2_bulk(a.w + (size_t)gv_row_of<EPI>(o, gt) * a.ldw, (uint32_t)a.k * 2u);
  }
  pdl_wait();
  trace_mark(trs, 2);
  uint64_t tag = 0;
  if constexpr (EPI == kGvLL)
    tag = (uint64_t)((uint32_t)(*(volatile const uint64_t*)a.epoch * a.tag_mult + a.tag_add)) << 32;

  float bv = -INFINITY;  // kGvArgmax: running best of this leader lane's (row, column) slot
  int bi = INT_MAX;
  const bool leader = (warp == grp * gw);
  for (int pass = 0; pass < passes; ++pass) {
    const int o0 = col_base + pass * sub_cols + grp * kOpg;
    const __nv_bfloat16* wr[kGvRows];
#pragma unroll
    for (int r = 0; r < kGvRows; ++r) {
      const int o = gv_out_of<EPI>(o0, r);
      wr[r] = a.w + (o < a.n_out ? (size_t)gv_row_of<EPI>(o, r) * a.ldw : 0);  // out of range: row 0, discarded
    }
    float acc[kGvRows][NB];
#pragma unroll
    for (int r = 0; r < kGvRows; ++r)
#pragma unroll
      for (int i = 0; i < NB; ++i) acc[r][i] = 0.f;
    int v = gt;
    for (; v + tk < nvec; v += 2 * tk) {
      uint4 w0[kGvRows], w1[kGvRows];
#pragma unroll
      for (int r = 0; r < kGvRows; ++r) {
        w0[r] = ld_stream16(wr[r] + (size_t)v * 8);
        w1[r] = ld_stream16(wr[r] + (size_t)(v + tk) * 8);
      }
      gv_fma<NB>(acc, w0, a, v);
      gv_fma<NB>(acc, w1, a, v + tk);
    }
    if (v < nvec) {
      uint4 w0[kGvRows];
#pragma unroll
      for (int r = 0; r < kGvRows; ++r) w0[r] = ld_stream16(wr[r] + (size_t)v * 8);
      gv_fma<NB>(acc, w0, a, v);
    }
    if (pass == passes - 1) pdl_launch_dependents();  // (every load of this CTA is issued)
#pragma unroll
    for (int r = 0; r < kGvRows; ++r)
#pragma unroll
      for (int i = 0; i < NB; ++i) acc[r][i] = warp_sum(acc[r][i]);
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < kGvRows; ++r)
#pragma unroll
        for (int i = 0; i < NB; ++i) red[warp][r * NB + i] = acc[r][i];
    }
    __syncthreads();
    if (leader) {
      if constexpr (EPI == kGvSilu) {
        if (lane < (kGvRows / 2) * NB) {
          const int j = lane / NB, i = lane % NB;
          float g = 0.f, u = 0.f;
          for (int w = 0; w < gw; ++w) {  // group warps in order: deterministic
            g += red[warp + w][(2 * j) * NB + i];
            u += red[warp + w][(2 * j + 1) * NB + i];
          }
          const int o = o0 + j;
          if (o < a.n_out && i < a.b) a.act[(size_t)i * a.ld_act + o] = f2bf(g / (1.f + __expf(-g)) * u);
        }
      } else {
        if (lane < kGvRows * NB) {
          const int r = lane / NB, i = lane % NB;
          float s = 0.f;
          for (int w = 0; w < gw; ++w) s += red[warp + w][lane];
          const int o = o0 + r;
          if (o < a.n_out && i < a.b) {
            if constexpr (EPI == kGvLL) {
              for (int d = 0; d < dst.n; ++d)
                st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(dst.p[d]) + (size_t)i * a.n_out + o,
                                   tag | __float_as_uint(s));
            } else {
              a.out[(size_t)i * a.n_out + o] = s;
              if constexpr (EPI == kGvArgmax) {
                const int ix = a.vocab0 + o;
                if (s > bv || (s == bv && ix < bi)) {
                  bv = s;
                  bi = ix;
                }
              }
            }
          }
        }
      }
    }
    __syncthreads();  // red[] is rewritten by the next pass
  }
  if constexpr (EPI == kGvArgmax) {
    if (leader && lane < kGvRows * NB) cs[grp][lane] = ArgmaxCand{bv, bi};
    __syncthreads();
    if (threadIdx.x < NB && (int)threadIdx.x < a.b) {
      const int i = threadIdx.x;
      float v = -INFINITY;
      int ix = INT_MAX;
      for (int g = 0; g < groups; ++g)
        for (int r = 0; r < kGvRows; ++r) {
          const ArgmaxCand c = cs[g][r * NB + i];
          if (c.val > v || (c.val == v && c.idx < ix)) {
            v = c.val;
            ix = c.idx;
          }
        }
      a.cand[(size_t)i * a.ntiles + blockIdx.x] = ArgmaxCand{v, ix};
    }
  }
  trace_mark(trs, 3);
}

// Row groups per CTA: the most (fewest lanes per row, most vectors in flight per thread) that
// still gives >= 2 CTAs per SM; then fewer lanes per row while more than half would idle.
int gv_groups(int n_out, int opg, int k) {
  const int nvec = k / 8;
  int groups = 1;
  for (int g = kGvWarps; g >= 1; g /= 2) {
    if ((n_out + opg * g - 1) / (opg * g) >= kGvTargetCtas) {
      groups = g;
      break;
    }
  }
  while (groups < kGvWarps && 32 * (kGvWarps / groups) > 2 * nvec) groups *= 2;
  return groups;
}

template <int EPI>
int gv_launch(GvArgs a, const DstList& dst, int grid, cudaStream_t st) {
  switch (a.b <= 1 ? 1 : (a.b <= 2 ? 2 : 4)) {
    case 1:
      return launch_k(gemv_kernel<1, EPI>, dim3(grid), dim3(kGvThreads), 0, st, true, a, dst);
    case 2:
      return launch_k(gemv_kernel<2, EPI>, dim3(grid), dim3(kGvThreads), 0, st, true, a, dst);
    default:
      return launch_k(gemv_kernel<4, EPI>, dim3(grid), dim3(kGvThreads), 0, st, true, a, dst);
  }
}

int gv_check(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx) {
  TPS_CHECK_ARG(w && x, "gemv: null operand");
  TPS_CHECK_ARG(b >= 1 && b <= kGvMaxB, "gemv: 1 <= b <= 4");
  TPS_CHECK_ARG(n >= 1 && n < INT_MAX / 2 && k >= 8 && k % 8 == 0 && k < INT_MAX / 2, "gemv: k % 8 == 0");
  TPS_CHECK_ARG(ldw >= k && ldw % 8 == 0 && ldx >= k && ldx % 8 == 0, "gemv: ldw, ldx >= k and % 8 == 0");
  TPS_CHECK_ARG((reinterpret_cast<uintptr_t>(w) & 15) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0,
                "gemv: operands must be 16-byte aligned");
  return kOk;
}

GvArgs gv_args(const void* w, int64_t n_out, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx) {
  GvArgs a = {};
  a.w = reinterpret_cast<const __nv_bfloat16*>(w);
  a.ldw = ldw;
  a.n_out = (int)n_out;
  a.k = (int)k;
  a.x = reinterpret_cast<const __nv_bfloat16*>(x);
  a.ldx = ldx;
  a.b = (int)b;
  return a;
}

}  // namespace

int gemv_max_rows() { return kGvMaxB; }

int trace_register_gemv(uint64_t* p, unsigned int* c, unsigned int n) { return trace_register(p, c, n); }

int gemv(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx, float* out,
         cudaStream_t st) {
  if (int e = gv_check(w, n, k, ldw, x, b, ldx)) return e;
  TPS_CHECK_ARG(out, "gemv: null output");
  GvArgs a = gv_args(w, n, k, ldw, x, b, ldx);
  a.out = out;
  const int groups = gv_groups((int)n, kGvRows, (int)k);
  a.group_warps = kGvWarps / groups;
  const int cols = kGvRows * groups;
  return gv_launch<kGvPartial>(a, DstList{}, (int)((n + cols - 1) / cols), st);
}

int gemv_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx, void* act,
              int64_t ld_act, cudaStream_t st) {
  if (int e = gv_check(w, n, k, ldw, x, b, ldx)) return e;
  TPS_CHECK_ARG(act && n % 128 == 0 && ld_act >= n / 2, "gemv_silu: n = 2F with F % 64 == 0, ld_act >= F");
  GvArgs a = gv_args(w, n / 2, k, ldw, x, b, ldx);
  a.act = reinterpret_cast<__nv_bfloat16*>(act);
  a.ld_act = ld_act;
  const int groups = gv_groups((int)(n / 2), kGvRows / 2, (int)k);
  a.group_warps = kGvWarps / groups;
  const int cols = (kGvRows / 2) * groups;
  return gv_launch<kGvSilu>(a, DstList{}, (int)((n / 2 + cols - 1) / cols), st);
}

int gemv_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                 const DstList& dst, const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add, cudaStream_t st) {
  if (int e = gv_check(w, n, k, ldw, x, b, ldx)) return e;
  TPS_CHECK_ARG(epoch && dst.n >= 1 && dst.n <= kMaxPeers, "gemv_push_ll: epoch and 1..8 destinations");
  for (int d = 0; d < dst.n; ++d)
    TPS_CHECK_ARG(dst.p[d] && (reinterpret_cast<uintptr_t>(dst.p[d]) & 7) == 0, "gemv_push_ll: 8-byte aligned slots");
  GvArgs a = gv_args(w, n, k, ldw, x, b, ldx);
  a.epoch = epoch;
  a.tag_mult = tag_mult;
  a.tag_add = tag_add;
  const int groups = gv_groups((int)n, kGvRows, (int)k);
  a.group_warps = kGvWarps / groups;
  const int cols = kGvRows * groups;
  return gv_launch<kGvLL>(a, dst, (int)((n + cols - 1) / cols), st);
}

int gemv_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                float* logits, void* cand, int vocab0, cudaStream_t st) {
  if (int e = gv_check(w, n, k, ldw, x, b, ldx)) return e;
  TPS_CHECK_ARG(logits && cand, "gemv_argmax: null output");
  GvArgs a = gv_args(w, n, k, ldw, x, b, ldx);
  a.out = logits;
  a.cand = reinterpret_cast<ArgmaxCand*>(cand);
  a.ntiles = (int)((n + 127) / 128);
  a.vocab0 = vocab0;
  a.group_warps = kGvWarps / gv_groups((int)n, kGvRows, (int)k);
  return gv_launch<kGvArgmax>(a, DstList{}, a.ntiles, st);
}

}  // namespace tps
