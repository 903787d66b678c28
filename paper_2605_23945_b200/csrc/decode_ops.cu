// Memory-bound decode-step kernels around the tcgen05 projections:
// embedding gather, residual add + RMSNorm (the consumer of O/down partials and
// of the TP allreduce), fused QKV bias + RoPE + paged-KV append, SiLU*up, the
// vocab-parallel greedy argmax with its cross-rank reduce, and the TP
// reduce-and-push (one-shot allreduce over NVLink P2P stores).
//
// Batch rows are indirected through row_slot[b] -> sample slot; per-slot state
// (position, page table, token history) stays where it is when the batch is
// compacted after completions, so a CUDA-graph replay only needs a new
// row_slot vector. row_slot[b] < 0 marks a padding row of a graph bucket.
#include "common.cuh"
#include "decode_ops.cuh"

namespace tps {

__device__ __forceinline__ void do_wait(const WaitSpec& w) {
  if (w.ctr == nullptr) return;
  if (threadIdx.x == 0) {
    const uint64_t target = w.add + (w.epoch ? (*(volatile const uint64_t*)w.epoch) * w.mult : 0ull);
    wait_counter_geq(w.ctr, target);
  }
  __syncthreads();
}

__device__ __forceinline__ void do_signal(const SignalSpec& s) {
  if (s.n == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's (possibly remote) stores are visible system-wide
    const unsigned int nblocks = gridDim.x * gridDim.y * gridDim.z;
    const unsigned int prev = atomicAdd(s.done, 1u);
    if (prev == nblocks - 1) {
      *s.done = 0u;  // re-arm for the next launch / graph replay
      __threadfence_system();
      for (int i = 0; i < s.n; ++i) red_release_sys_add(s.ctr[i], 1ull);
    }
  }
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
                             const int* __restrict__ history, int hist_ld,
                             const __nv_bfloat16* __restrict__ table, int H,
                             float* __restrict__ resid) {
  const int b = blockIdx.x;
  const int slot = row_slot[b];
  int tok = 0;
  if (slot >= 0) tok = history[(size_t)slot * hist_ld + pos_by_slot[slot]];
  const __nv_bfloat162* src = reinterpret_cast<const __nv_bfloat162*>(table + (size_t)tok * H);
  float2* dst = reinterpret_cast<float2*>(resid + (size_t)b * H);
  for (int i = threadIdx.x; i < H / 2; i += blockDim.x) dst[i] = __bfloat1622float2(src[i]);
}

// ------------------------------------------------- residual add + RMSNorm ---
// resid[b] += sum_i src_i[b] (list order); out[b] = bf16(resid * rstd * w)
constexpr int kNormThreads = 256;
__global__ void __launch_bounds__(kNormThreads) add_norm_kernel(
    float* __restrict__ resid, SrcList src, WaitSpec wait, const __nv_bfloat16* __restrict__ w,
    float eps, int H, __nv_bfloat16* __restrict__ out, int ldo) {
  __shared__ float red[32];
  const int b = blockIdx.x;
  do_wait(wait);
  float4* r4 = reinterpret_cast<float4*>(resid + (size_t)b * H);
  const int H4 = H / 4;
  float ss = 0.f;
  for (int i = threadIdx.x; i < H4; i += kNormThreads) {
    float4 v = r4[i];
    for (int s = 0; s < src.n; ++s) {
      const float4 p = reinterpret_cast<const float4*>(src.p[s] + (size_t)b * H)[i];
      v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
    }
    r4[i] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = block_sum<kNormThreads>(ss, red);
  const float rstd = rsqrtf(ss / (float)H + eps);
  __nv_bfloat16* o = out + (size_t)b * ldo;
  for (int i = threadIdx.x; i < H4; i += kNormThreads) {
    const float4 v = r4[i];
    const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(w) + 2 * i;
    const float2 w01 = __bfloat1622float2(wp[0]);
    const float2 w23 = __bfloat1622float2(wp[1]);
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(o) + 2 * i;
    op[0] = __floats2bfloat162_rn(v.x * rstd * w01.x, v.y * rstd * w01.y);
    op[1] = __floats2bfloat162_rn(v.z * rstd * w23.x, v.w * rstd * w23.y);
  }
}

// ------------------------------------------- TP one-shot allreduce (push) ---
// Sum this rank's split-K partials and store the [rows][cols] result into this
// rank's slot of every TP peer's receive area (NVLink P2P stores), then signal.
constexpr int kPushBlocks = 64;
__global__ void __launch_bounds__(256) reduce_push_kernel(SrcList src, DstList dst, int64_t n4,
                                                          SignalSpec sig) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(src.p[0])[i];
    for (int s = 1; s < src.n; ++s) {
      const float4 p = reinterpret_cast<const float4*>(src.p[s])[i];
      v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
    }
    for (int d = 0; d < dst.n; ++d) reinterpret_cast<float4*>(dst.p[d])[i] = v;
  }
  do_signal(sig);
}

// ---------------------------------------------- QKV bias + RoPE + KV append ---
// partial layout [split][B][Nqkv] with Nqkv = (nq + 2 nkv) * D, rows ordered
// [q heads | k heads | v heads] (canonical shard layout). RoPE is the
// rotate-half form used by Llama/Qwen2 with a host-built fp32 cos/sin table.
// KV cache per layer: [num_pages][nkv][P][D] bf16.
__global__ void qkv_rope_append_kernel(SrcList src, const __nv_bfloat16* __restrict__ bias,
                                       const int* __restrict__ row_slot,
                                       const int* __restrict__ pos_by_slot,
                                       const int* __restrict__ page_table, int max_pages,
                                       const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                       int B, int nq, int nkv, int D, int P,
                                       __nv_bfloat16* __restrict__ q_out,
                                       __nv_bfloat16* __restrict__ k_cache,
                                       __nv_bfloat16* __restrict__ v_cache) {
  const int b = blockIdx.x;
  const int h = blockIdx.y;
  const int i = threadIdx.x;  // 0 .. D/2-1
  const int half = D / 2;
  const int slot = row_slot[b];
  const int N = (nq + 2 * nkv) * D;
  const int pos = slot >= 0 ? pos_by_slot[slot] : 0;
  auto val = [&](int c) {
    float v = bias ? bf2f(bias[c]) : 0.f;
    for (int s = 0; s < src.n; ++s) v += src.p[s][(size_t)b * N + c];
    return v;
  };
  const float cs = cos_t[(size_t)pos * half + i];
  const float sn = sin_t[(size_t)pos * half + i];
  if (h < nq) {
    const int c0 = h * D;
    const float x1 = val(c0 + i), x2 = val(c0 + i + half);
    __nv_bfloat16* q = q_out + ((size_t)b * nq + h) * D;
    q[i] = f2bf(x1 * cs - x2 * sn);
    q[i + half] = f2bf(x2 * cs + x1 * sn);
    return;
  }
  if (slot < 0) return;
  const int j = h - nq;
  const int kc0 = nq * D + j * D;
  const int vc0 = (nq + nkv) * D + j * D;
  const float k1 = val(kc0 + i), k2 = val(kc0 + i + half);
  const float v1 = val(vc0 + i), v2 = val(vc0 + i + half);
  const int page = page_table[(size_t)slot * max_pages + pos / P];
  const size_t off = (((size_t)page * nkv + j) * P + (pos % P)) * D;
  k_cache[off + i] = f2bf(k1 * cs - k2 * sn);
  k_cache[off + i + half] = f2bf(k2 * cs + k1 * sn);
  v_cache[off + i] = f2bf(v1);
  v_cache[off + i + half] = f2bf(v2);
}

// ------------------------------------------------------------- SiLU * up ---
// partial layout [split][B][2F] = [gate rows | up rows]; out[b][f] = bf16(silu(g) * u)
__global__ void silu_mul_kernel(SrcList src, int B, int F, __nv_bfloat16* __restrict__ out, int ldo) {
  const int64_t total = (int64_t)B * F;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(t / F), f = (int)(t % F);
    float g = 0.f, u = 0.f;
    for (int s = 0; s < src.n; ++s) {
      const float* p = src.p[s] + (size_t)b * 2 * F;
      g += p[f];
      u += p[F + f];
    }
    const float sg = g / (1.f + __expf(-g));
    out[(size_t)b * ldo + f] = f2bf(sg * u);
  }
}

// ------------------------------------------------------- greedy argmax ---
// Stage 1: per (row, vocab chunk) max with the smallest index on ties.
constexpr int kArgmaxThreads = 256;
__device__ __forceinline__ void cand_merge(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__global__ void __launch_bounds__(kArgmaxThreads) argmax_stage1_kernel(
    SrcList src, int B, int V, int vocab_offset, int nchunk, ArgmaxCand* __restrict__ cand,
    SignalSpec sig) {
  __shared__ float sv[kArgmaxThreads / 32];
  __shared__ int si[kArgmaxThreads / 32];
  const int b = blockIdx.x, c = blockIdx.y;
  const int per = (V + nchunk - 1) / nchunk;
  const int lo = c * per, hi = min(V, lo + per);
  float best = -INFINITY;
  int bidx = 0x7fffffff;
  for (int j = lo + threadIdx.x; j < hi; j += kArgmaxThreads) {
    float v = 0.f;
    for (int s = 0; s < src.n; ++s) v += src.p[s][(size_t)b * V + j];
    cand_merge(best, bidx, v, j + vocab_offset);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
    cand_merge(best, bidx, v2, i2);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sv[w] = best; si[w] = bidx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kArgmaxThreads / 32; ++k) cand_merge(best, bidx, sv[k], si[k]);
    cand[(size_t)b * nchunk + c] = ArgmaxCand{best, bidx};
  }
  do_signal(sig);
}

// Stage 2: reduce the candidates of every TP rank (list order = rank order),
// append the token to the sample's history and advance its position.
__global__ void argmax_finalize_kernel(CandList cands, int nchunk, WaitSpec wait,
                                       const int* __restrict__ row_slot, int* __restrict__ pos_by_slot,
                                       const int* __restrict__ prompt_len, int* __restrict__ history,
                                       int hist_ld, int* __restrict__ out_tok) {
  const int b = blockIdx.x;
  do_wait(wait);
  float best = -INFINITY;
  int bidx = 0x7fffffff;
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
}

__global__ void epoch_advance_kernel(uint64_t* epoch) { *epoch += 1ull; }

// Plain fp32 sum of a SrcList into a dense buffer (tests / logits export).
__global__ void sum_src_kernel(SrcList src, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int s = 0; s < src.n; ++s) v += src.p[s][i];
    out[i] = v;
  }
}

// -------------------------------------------------------------- launchers ---
int embed(const int* row_slot, const int* pos_by_slot, const int* history, int hist_ld,
          const void* table, int H, int B, float* resid, cudaStream_t st) {
  TPS_CHECK_ARG(H % 2 == 0 && B > 0, "embed: H must be even, B > 0");
  embed_kernel<<<B, 256, 0, st>>>(row_slot, pos_by_slot, history, hist_ld,
                                  reinterpret_cast<const __nv_bfloat16*>(table), H, resid);
  TPS_LAUNCH_CHECK();
  return kOk;
}

int add_norm(float* resid, const SrcList& src, const WaitSpec& wait, const void* w, float eps, int H,
             int B, void* out, int ldo, cudaStream_t st) {
  TPS_CHECK_ARG(H % 4 == 0 && ldo % 4 == 0 && B > 0, "add_norm: H, ldo must be multiples of 4");
  TPS_CHECK_ARG(src.n >= 0 && src.n <= kMaxSrc, "add_norm: too many sources");
  add_norm_kernel<<<B, kNormThreads, 0, st>>>(resid, src, wait, reinterpret_cast<const __nv_bfloat16*>(w),
                                              eps, H, reinterpret_cast<__nv_bfloat16*>(out), ldo);
  TPS_LAUNCH_CHECK();
  return kOk;
}

int reduce_push(const SrcList& src, const DstList& dst, int64_t n, const SignalSpec& sig, cudaStream_t st) {
  TPS_CHECK_ARG(n % 4 == 0 && src.n >= 1 && dst.n >= 1, "reduce_push: n % 4 == 0, >=1 src/dst");
  reduce_push_kernel<<<kPushBlocks, 256, 0, st>>>(src, dst, n / 4, sig);
  TPS_LAUNCH_CHECK();
  return kOk;
}

int qkv_rope_append(const SrcList& src, const void* bias, const int* row_slot, const int* pos_by_slot,
                    const int* page_table, int max_pages, const float* cos_t, const float* sin_t, int B,
                    int nq, int nkv, int D, int P, void* q_out, void* k_cache, void* v_cache,
                    cudaStream_t st) {
  TPS_CHECK_ARG(D % 2 == 0 && D <= 256 && B > 0 && nq > 0 && nkv > 0, "qkv_rope_append: bad shape");
  dim3 grid(B, nq + nkv);
  qkv_rope_append_kernel<<<grid, D / 2, 0, st>>>(
      src, reinterpret_cast<const __nv_bfloat16*>(bias), row_slot, pos_by_slot, page_table, max_pages,
      cos_t, sin_t, B, nq, nkv, D, P, reinterpret_cast<__nv_bfloat16*>(q_out),
      reinterpret_cast<__nv_bfloat16*>(k_cache), reinterpret_cast<__nv_bfloat16*>(v_cache));
  TPS_LAUNCH_CHECK();
  return kOk;
}

int silu_mul(const SrcList& src, int B, int F, void* out, int ldo, cudaStream_t st) {
  TPS_CHECK_ARG(B > 0 && F > 0, "silu_mul: bad shape");
  const int64_t total = (int64_t)B * F;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
  silu_mul_kernel<<<blocks, 256, 0, st>>>(src, B, F, reinterpret_cast<__nv_bfloat16*>(out), ldo);
  TPS_LAUNCH_CHECK();
  return kOk;
}

int argmax_stage1(const SrcList& src, int B, int V, int vocab_offset, int nchunk, void* cand,
                  const SignalSpec& sig, cudaStream_t st) {
  TPS_CHECK_ARG(B > 0 && V > 0 && nchunk > 0, "argmax_stage1: bad shape");
  dim3 grid(B, nchunk);
  argmax_stage1_kernel<<<grid, kArgmaxThreads, 0, st>>>(src, B, V, vocab_offset, nchunk,
                                                        reinterpret_cast<ArgmaxCand*>(cand), sig);
  TPS_LAUNCH_CHECK();
  return kOk;
}

int argmax_finalize(const CandList& cands, int nchunk, const WaitSpec& wait, int B, const int* row_slot,
                    int* pos_by_slot, const int* prompt_len, int* history, int hist_ld, int* out_tok,
                    cudaStream_t st) {
  TPS_CHECK_ARG(B > 0 && cands.n >= 1 && cands.n <= kMaxPeers, "argmax_finalize: bad args");
  argmax_finalize_kernel<<<B, 32, 0, st>>>(cands, nchunk, wait, row_slot, pos_by_slot, prompt_len, history,
                                           hist_ld, out_tok);
  TPS_LAUNCH_CHECK();
  return kOk;
}

int epoch_advance(uint64_t* epoch, cudaStream_t st) {
  epoch_advance_kernel<<<1, 1, 0, st>>>(epoch);
  TPS_LAUNCH_CHECK();
  return kOk;
}

int sum_src(const SrcList& src, int64_t n, float* out, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
  if (blocks < 1) blocks = 1;
  sum_src_kernel<<<blocks, 256, 0, st>>>(src, n, out);
  TPS_LAUNCH_CHECK();
  return kOk;
}

}  // namespace tps
