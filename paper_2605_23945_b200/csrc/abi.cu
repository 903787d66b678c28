// extern "C" entry points of libtpshift_b200.so (declared in include/tpshift_b200.h).
// Each one validates its arguments, packs host pointer lists into by-value
// kernel parameter structs and forwards to the kernel launchers.
#include <stdio.h>

#include <string>
#include <vector>

#include "../../include/tpshift_b200.h"
#include "common.cuh"
#include "decode_ops.cuh"

namespace tps {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// launchers (defined in the kernel translation units)
void set_pdl(bool on);
int linear_splits(int64_t n, int64_t k, int64_t b);
int linear_push(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                int64_t ldx, const DstList& dst, int64_t split_stride, int splits, const SignalSpec& sig,
                cudaStream_t stream);
int linear_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                int64_t ldx, void* act, int64_t ld_act, cudaStream_t stream);
int linear(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
           int64_t ldx, float* out, int splits, cudaStream_t stream);
int cluster_splits(int64_t n, int64_t k, int64_t b);
int linear_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                  int64_t ldx, float* logits, void* cand, int vocab0, cudaStream_t stream);
int linear_push_ll_cluster(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                           int64_t x_rows, int64_t ldx, const DstList& dst, const uint64_t* tag_epoch,
                           uint32_t tag_mult, uint32_t tag_add, cudaStream_t stream);
int gemv_max_rows();
int gemv(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx, float* out,
         cudaStream_t st);
int gemv_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx, void* act,
              int64_t ld_act, cudaStream_t st);
int gemv_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                 const DstList& dst, const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add, cudaStream_t st);
int gemv_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                float* logits, void* cand, int vocab0, cudaStream_t st);
int embed(const int*, const int*, const int*, const int*, int, const void*, int, int, float*, cudaStream_t);
int add_norm(float*, const Src&, const WaitSpec&, const void*, float, int, int, void*, int, cudaStream_t);
int reduce_push(const Src&, const DstList&, long long, const SignalSpec&, cudaStream_t);
int qkv_rope_append(const Src&, const void*, const int*, const int*, const int*, const int*, int, const float*,
                    const float*, int, int, int, int, int, void*, void*, void*, cudaStream_t);
int silu_mul(const Src&, int, int, void*, int, cudaStream_t);
int argmax_stage1(const Src&, int, int, int, int, void*, const SignalSpec&, cudaStream_t,
                  const SamplerSpec* smp = nullptr);
int argmax_finalize(const CandList&, int, const WaitSpec&, int, const int*, int*, const int*, int*, int, int*,
                    cudaStream_t);
int epoch_advance(uint64_t*, cudaStream_t);
int sum_src(const Src&, long long, float*, cudaStream_t);
int attn_splits(int B, int nkv, int max_pages);
int attn_balanced_grid(int D);
int paged_attention(const void*, const void*, const void*, const int*, const int*, const int*, const int*, int,
                    int, int, int, int, int, float*, float*, float*, unsigned int*, void*, const Src&, const void*,
                    const float*, const float*, cudaStream_t);
int copy_items(const void*, int, int, int, cudaStream_t);
int kv_move_items(const void*, int, int64_t, void*, int, int, int64_t, void*, int*, cudaStream_t);
int prefill_group_positions(int G);
int paged_prefill_attention(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                            const int* row_pos, const int* grp_rows, const int* grp_n, int max_groups,
                            const int* page_table, int max_pages, int nq, int nkv, int D, void* out,
                            cudaStream_t st);
int configure_gemm();
int configure_attention();
int configure_copy();
int configure_decode_ops();
int configure_persist();
int reduce_push_ll(const Src& src, const DstList& dst, long long n, const uint64_t* epoch, uint32_t mult,
                   uint32_t add, cudaStream_t st);
int linear_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                   int64_t ldx, const DstList& dst, int64_t split_stride, int splits, const uint64_t* tag_epoch,
                   uint32_t tag_mult, uint32_t tag_add, cudaStream_t stream);
int add_norm_ll(float* resid, const uint64_t* ll, int nsrc, long long stride, const uint64_t* epoch, uint32_t mult,
                uint32_t add, const void* w, float eps, int H, int B, void* out, int ldo, uint64_t* ctr,
                uint64_t bump, cudaStream_t st);
int trace_register_decode(uint64_t*, unsigned int*, unsigned int);
int trace_register_attention(uint64_t*, unsigned int*, unsigned int);
int trace_register_attention_bal(uint64_t*, unsigned int*, unsigned int);
int trace_register_gemm(uint64_t*, unsigned int*, unsigned int);
int trace_register_attention_prefill(uint64_t*, unsigned int*, unsigned int);
int trace_register_gemv(uint64_t*, unsigned int*, unsigned int);
int barrier(uint64_t* const*, int, const uint64_t*, int, int, uint64_t, cudaStream_t);
int ipc_get_handle(const void*, void*, int64_t*);
int ipc_open(const void*, void**);
int ipc_close(void*);

static int make_src(const float* base, int n, int64_t stride, Src* out) {
  if (n < 0 || n > 1024) return fail(kInvalid, "source count must be in [0, 1024]");
  if (n > 0 && !base) return fail(kInvalid, "null source base");
  out->base = base;
  out->n = n;
  out->stride = stride;
  return kOk;
}

static int make_sig(uint64_t* const* ctrs, int n, unsigned int* done, SignalSpec* out) {
  if (n < 0 || n > kMaxPeers) return fail(kInvalid, "signal list longer than 8 entries");
  if (n > 0 && !done) return fail(kInvalid, "signal list needs a done counter");
  out->n = n;
  out->done = done;
  for (int i = 0; i < n; ++i) out->ctr[i] = ctrs[i];
  return kOk;
}

static WaitSpec make_wait(const tps_wait* w) {
  WaitSpec s{};
  if (w) {
    s.ctr = w->ctr;
    s.epoch = w->epoch;
    s.mult = w->mult;
    s.add = w->add;
  }
  return s;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- soft-abort word (common.cuh): one host-mapped word per process, its device address
// installed in every translation unit's copy of g_abort_word on every initialised device
static std::vector<AbortSetter>& abort_setters() {
  static std::vector<AbortSetter> v;
  return v;
}
int register_abort_setter(AbortSetter f) {
  abort_setters().push_back(f);
  return (int)abort_setters().size();
}
static unsigned int* g_abort_host = nullptr;

static int install_abort_word(int device) {
  // Best effort: without the word a fired watchdog still abandons its wait (it only cannot
  // tell the other waits or the host), so a failure here must not fail tps_init.
  static std::vector<int> done;  // devices whose translation units hold the pointer already
  for (int d : done)
    if (d == device) return kOk;
  if (!g_abort_host) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return kOk;
    }
    g_abort_host = static_cast<unsigned int*>(p);
    *reinterpret_cast<volatile unsigned int*>(g_abort_host) = 0u;
  }
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, g_abort_host, 0) != cudaSuccess) {
    cudaGetLastError();
    return kOk;
  }
  for (AbortSetter f : abort_setters())
    if (f(static_cast<unsigned int*>(dptr)) != 0) cudaGetLastError();
  done.push_back(device);
  return kOk;
}

}  // namespace tps

using namespace tps;

extern "C" {

const char* tps_version(void) { return "tpshift_b200 1.1 (sm_100a; tcgen05 GEMM, paged GQA decode, P2P switch, PDL)"; }

const char* tps_last_error(void) { return g_last_error.c_str(); }

unsigned int tps_abort_status(void) {
  return g_abort_host ? *reinterpret_cast<volatile unsigned int*>(g_abort_host) : 0u;
}

void tps_abort_clear(void) {
  if (g_abort_host) *reinterpret_cast<volatile unsigned int*>(g_abort_host) = 0u;
}

int tps_init(int device, int* sm_count) {
  TPS_CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  TPS_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (prop.major != 10)
    return fail(kUnsupported, std::string("libtpshift_b200 is built for sm_100a; device is sm_") +
                                  std::to_string(prop.major) + std::to_string(prop.minor));
  // kernel attributes (dynamic smem opt-in) are set once here, outside any stream capture
  int rc = configure_gemm();
  if (!rc) rc = configure_attention();
  if (!rc) rc = configure_copy();
  if (!rc) rc = configure_decode_ops();
  if (!rc) rc = configure_persist();
  if (!rc) rc = install_abort_word(device);
  return rc;
}

void tps_set_pdl(int on) { set_pdl(on != 0); }

int tps_linear_splits(int64_t n, int64_t k, int64_t b) { return linear_splits(n, k, b); }

int tps_linear(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
               int64_t ldx, float* out, int splits, void* stream) {
  return linear(w, n, k, ldw, x, b, x_rows, ldx, out, splits, S(stream));
}

int tps_linear_push(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                    int64_t ldx, float* const* dsts, int ndst, int64_t split_stride, int splits,
                    uint64_t* const* sig_ctrs, int nsig, unsigned int* done, void* stream) {
  TPS_CHECK_ARG(ndst >= 1 && ndst <= kMaxPeers && dsts, "linear_push: 1..8 destinations");
  DstList dl;
  dl.n = ndst;
  for (int i = 0; i < ndst; ++i) dl.p[i] = dsts[i];
  SignalSpec sg;
  int rc = make_sig(sig_ctrs, nsig, done, &sg);
  if (rc) return rc;
  return linear_push(w, n, k, ldw, x, b, x_rows, ldx, dl, split_stride, splits, sg, S(stream));
}

int tps_linear_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                       int64_t ldx, uint64_t* const* dsts, int ndst, int64_t split_stride, int splits,
                       const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add, void* stream) {
  TPS_CHECK_ARG(ndst >= 1 && ndst <= kMaxPeers && dsts, "linear_push_ll: 1..8 destinations");
  DstList dl;
  dl.n = ndst;
  for (int i = 0; i < ndst; ++i) dl.p[i] = reinterpret_cast<float*>(dsts[i]);
  return linear_push_ll(w, n, k, ldw, x, b, x_rows, ldx, dl, split_stride, splits, epoch, tag_mult, tag_add,
                        S(stream));
}

int tps_add_norm_ll(float* resid, const uint64_t* ll, int nsrc, int64_t stride, const uint64_t* epoch,
                    uint32_t tag_mult, uint32_t tag_add, const void* w, float eps, int H, int B, void* out, int ldo,
                    uint64_t* ctr, uint64_t bump, void* stream) {
  TPS_CHECK_ARG(resid && w && out, "add_norm_ll: null pointer");
  return add_norm_ll(resid, ll, nsrc, stride, epoch, tag_mult, tag_add, w, eps, H, B, out, ldo, ctr, bump,
                     S(stream));
}

int tps_linear_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                    int64_t ldx, void* act, int64_t ld_act, void* stream) {
  return linear_silu(w, n, k, ldw, x, b, x_rows, ldx, act, ld_act, S(stream));
}

int tps_cluster_splits(int64_t n, int64_t k, int64_t b) { return cluster_splits(n, k, b); }

int tps_gemv_max_rows(void) { return gemv_max_rows(); }

int tps_gemv(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx, float* out,
             void* stream) {
  return gemv(w, n, k, ldw, x, b, ldx, out, S(stream));
}

int tps_gemv_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx, void* act,
                  int64_t ld_act, void* stream) {
  return gemv_silu(w, n, k, ldw, x, b, ldx, act, ld_act, S(stream));
}

int tps_gemv_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                     uint64_t* const* dsts, int ndst, const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add,
                     void* stream) {
  TPS_CHECK_ARG(ndst >= 1 && ndst <= kMaxPeers && dsts, "gemv_push_ll: 1..8 destinations");
  DstList dl;
  dl.n = ndst;
  for (int i = 0; i < ndst; ++i) dl.p[i] = reinterpret_cast<float*>(dsts[i]);
  return gemv_push_ll(w, n, k, ldw, x, b, ldx, dl, epoch, tag_mult, tag_add, S(stream));
}

int tps_gemv_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                    float* logits, void* cand, int vocab0, void* stream) {
  return gemv_argmax(w, n, k, ldw, x, b, ldx, logits, cand, vocab0, S(stream));
}


int tps_linear_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                      int64_t ldx, float* logits, void* cand, int vocab0, void* stream) {
  return linear_argmax(w, n, k, ldw, x, b, x_rows, ldx, logits, cand, vocab0, S(stream));
}

int tps_linear_push_ll_cluster(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                               int64_t x_rows, int64_t ldx, uint64_t* const* dsts, int ndst, const uint64_t* epoch,
                               uint32_t tag_mult, uint32_t tag_add, void* stream) {
  TPS_CHECK_ARG(ndst >= 1 && ndst <= kMaxPeers && dsts, "linear_push_ll_cluster: 1..8 destinations");
  DstList dl;
  dl.n = ndst;
  for (int i = 0; i < ndst; ++i) dl.p[i] = reinterpret_cast<float*>(dsts[i]);
  return linear_push_ll_cluster(w, n, k, ldw, x, b, x_rows, ldx, dl, epoch, tag_mult, tag_add, S(stream));
}

int tps_prefill_group_positions(int G) { return prefill_group_positions(G); }

int tps_prefill_attention(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                          const int* row_pos, const int* grp_rows, const int* grp_n, int max_groups,
                          const int* page_table, int max_pages, int nq, int nkv, int D, void* out, void* stream) {
  TPS_CHECK_ARG(q && k_cache && v_cache && row_slot && row_pos && grp_rows && grp_n && page_table && out,
                "prefill_attention: null pointer");
  return paged_prefill_attention(q, k_cache, v_cache, row_slot, row_pos, grp_rows, grp_n, max_groups, page_table,
                                 max_pages, nq, nkv, D, out, S(stream));
}

int tps_embed(const int* row_slot, const int* pos_by_slot, const int* row_pos, const int* history, int hist_ld,
              const void* table, int H, int B, float* resid, void* stream) {
  TPS_CHECK_ARG(row_slot && pos_by_slot && history && table && resid, "embed: null pointer");
  return embed(row_slot, pos_by_slot, row_pos, history, hist_ld, table, H, B, resid, S(stream));
}

int tps_add_norm(float* resid, const float* src, int nsrc, int64_t src_stride, const tps_wait* wait,
                 const void* w, float eps, int H, int B, void* out, int ldo, void* stream) {
  TPS_CHECK_ARG(resid && w && out, "add_norm: null pointer");
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  return add_norm(resid, s, make_wait(wait), w, eps, H, B, out, ldo, S(stream));
}

int tps_reduce_push_ll(const float* src, int nsrc, int64_t src_stride, uint64_t* const* dsts, int ndst, int64_t n,
                       const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add, void* stream) {
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  TPS_CHECK_ARG(ndst >= 1 && ndst <= kMaxPeers && dsts, "reduce_push_ll: 1..8 destinations");
  DstList dl;
  dl.n = ndst;
  for (int i = 0; i < ndst; ++i) {
    TPS_CHECK_ARG((reinterpret_cast<uintptr_t>(dsts[i]) & 31) == 0, "reduce_push_ll: 32B-aligned destinations");
    dl.p[i] = reinterpret_cast<float*>(dsts[i]);
  }
  return reduce_push_ll(s, dl, n, epoch, tag_mult, tag_add, S(stream));
}

int tps_reduce_push(const float* src, int nsrc, int64_t src_stride, float* const* dsts, int ndst, int64_t n,
                    uint64_t* const* sig_ctrs, int nsig, unsigned int* done, void* stream) {
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  TPS_CHECK_ARG(ndst >= 1 && ndst <= kMaxPeers && dsts, "reduce_push: 1..8 destinations");
  DstList dl;
  dl.n = ndst;
  for (int i = 0; i < ndst; ++i) dl.p[i] = dsts[i];
  SignalSpec sg;
  rc = make_sig(sig_ctrs, nsig, done, &sg);
  if (rc) return rc;
  return reduce_push(s, dl, n, sg, S(stream));
}

int tps_qkv_rope_append(const float* src, int nsrc, int64_t src_stride, const void* bias, const int* row_slot,
                        const int* pos_by_slot, const int* row_pos, const int* page_table, int max_pages,
                        const float* cos_t,
                        const float* sin_t, int B, int nq, int nkv, int D, int page_size, void* q_out,
                        void* k_cache, void* v_cache, void* stream) {
  TPS_CHECK_ARG(page_size == 64, "qkv_rope_append: page_size must be 64");
  TPS_CHECK_ARG(row_slot && pos_by_slot && page_table && cos_t && sin_t && q_out && k_cache && v_cache,
                "qkv_rope_append: null pointer");
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  return qkv_rope_append(s, bias, row_slot, pos_by_slot, row_pos, page_table, max_pages, cos_t, sin_t, B, nq, nkv,
                         D,
                         page_size, q_out, k_cache, v_cache, S(stream));
}

int tps_attn_splits(int B, int nkv, int max_pages) { return attn_splits(B, nkv, max_pages); }

int64_t tps_attn_workspace(int B, int nq, int D, int nsplit) {
  if (nsplit > 0) return (int64_t)B * nq * nsplit * D;
  return (int64_t)attn_balanced_grid(D) * 2 * 16 * D;
}

int tps_paged_attention(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                        const int* pos_by_slot, const int* row_pos, const int* page_table, int max_pages,
                        int B, int nq, int nkv, int D,
                        int nsplit, float* part_m, float* part_l, float* part_o, unsigned int* merge_ctr,
                        void* out, const float* qkv, int nqkv, int64_t qkv_stride, const void* qkv_bias,
                        const float* cos_t, const float* sin_t, void* stream) {
  TPS_CHECK_ARG(k_cache && v_cache && row_slot && pos_by_slot && page_table && part_m && part_l && part_o &&
                    merge_ctr && out && (q || qkv),
                "paged_attention: null pointer");
  Src s;
  int rc = make_src(qkv, qkv ? nqkv : 0, qkv_stride, &s);
  if (rc) return rc;
  return paged_attention(q, k_cache, v_cache, row_slot, pos_by_slot, row_pos, page_table, max_pages, B, nq,
                         nkv, D,
                         nsplit, part_m, part_l, part_o, merge_ctr, out, s, qkv_bias, cos_t, sin_t, S(stream));
}

int tps_silu_mul(const float* src, int nsrc, int64_t src_stride, int B, int F, void* out, int ldo, void* stream) {
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  return silu_mul(s, B, F, out, ldo, S(stream));
}

int tps_argmax_stage1(const float* src, int nsrc, int64_t src_stride, int B, int V, int vocab_offset, int nchunk,
                      void* cand, uint64_t* const* sig_ctrs, int nsig, unsigned int* done, void* stream) {
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  SignalSpec sg;
  rc = make_sig(sig_ctrs, nsig, done, &sg);
  if (rc) return rc;
  return argmax_stage1(s, B, V, vocab_offset, nchunk, cand, sg, S(stream));
}

int tps_sample_stage1(const float* src, int nsrc, int64_t src_stride, int B, int V, int vocab_offset, int nchunk,
                      void* cand, uint64_t* const* sig_ctrs, int nsig, unsigned int* done, const uint64_t* seeds,
                      const int* row_slot, const int* pos_by_slot, const int* row_pos, float temperature,
                      void* stream) {
  TPS_CHECK_ARG(seeds && row_slot && (pos_by_slot || row_pos), "sample_stage1: null sampler state");
  TPS_CHECK_ARG(temperature > 0.f, "sample_stage1: temperature must be > 0 (greedy: tps_argmax_stage1)");
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  SignalSpec sg;
  rc = make_sig(sig_ctrs, nsig, done, &sg);
  if (rc) return rc;
  SamplerSpec smp{seeds, row_slot, pos_by_slot, row_pos, 1.f / temperature};
  return argmax_stage1(s, B, V, vocab_offset, nchunk, cand, sg, S(stream), &smp);
}

int tps_argmax_finalize(const void* const* cands, int ncand, int nchunk, const tps_wait* wait, int B,
                        const int* row_slot, int* pos_by_slot, const int* prompt_len, int* history, int hist_ld,
                        int* out_tok, void* stream) {
  TPS_CHECK_ARG(ncand >= 1 && ncand <= kMaxPeers && cands, "argmax_finalize: 1..8 candidate arrays");
  CandList cl;
  cl.n = ncand;
  for (int i = 0; i < ncand; ++i) cl.p[i] = reinterpret_cast<const ArgmaxCand*>(cands[i]);
  return argmax_finalize(cl, nchunk, make_wait(wait), B, row_slot, pos_by_slot, prompt_len, history, hist_ld,
                         out_tok, S(stream));
}

int tps_epoch_advance(uint64_t* epoch, void* stream) {
  TPS_CHECK_ARG(epoch, "epoch_advance: null pointer");
  return epoch_advance(epoch, S(stream));
}

int tps_sum_partials(const float* src, int nsrc, int64_t src_stride, int64_t n, float* out, void* stream) {
  Src s;
  int rc = make_src(src, nsrc, src_stride, &s);
  if (rc) return rc;
  return sum_src(s, n, out, S(stream));
}

int tps_copy_items(const tps_copy_item* items, int n, int mode, int grid, void* stream) {
  static_assert(sizeof(tps_copy_item) == 32, "copy item layout");
  return copy_items(items, n, mode, grid, S(stream));
}

int tps_kv_move_items(const tps_kv_move* moves, int n_moves, int64_t n_items, void* dst_kv, int dst_num_pages,
                      int dst_nkv, int64_t chunk_bytes, tps_copy_item* items_out, int* bad_pages, void* stream) {
  static_assert(sizeof(tps_kv_move) == 56, "kv move layout");
  return kv_move_items(moves, n_moves, n_items, dst_kv, dst_num_pages, dst_nkv, chunk_bytes, items_out, bad_pages,
                       S(stream));
}

int tps_barrier(uint64_t* const* peer_slots, int npeers, const uint64_t* my_slots, int nslots, int self_slot,
                uint64_t epoch, void* stream) {
  return barrier(peer_slots, npeers, my_slots, nslots, self_slot, epoch, S(stream));
}

int tps_ipc_get_handle(const void* ptr, void* handle_out, int64_t* offset_out) {
  return ipc_get_handle(ptr, handle_out, offset_out);
}
int tps_ipc_open(const void* handle, void** base_out) { return ipc_open(handle, base_out); }
int tps_ipc_close(void* base) { return ipc_close(base); }

int tps_trace_enable(uint64_t* records, unsigned int* counter, unsigned int capacity) {
  TPS_CHECK_ARG((records && counter) || (!records && !counter), "trace: records and counter together");
  if (trace_register_decode(records, counter, capacity) || trace_register_attention(records, counter, capacity) ||
      trace_register_attention_bal(records, counter, capacity) || trace_register_gemm(records, counter, capacity) ||
      trace_register_attention_prefill(records, counter, capacity) || trace_register_gemv(records, counter, capacity))
    return fail(kCuda, "trace: cudaMemcpyToSymbol failed");
  return kOk;
}

}  // extern "C"
