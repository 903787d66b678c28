/*
 * tpshift_b200.h -- C ABI of libtpshift_b200.so, the B200 (sm_100a) execution
 * engine behind PAT's generation hot path (arXiv 2605.23945).
 *
 * The reference (`tpshift`, /root/reference/pkg) is a pure-Python simulator: it
 * has no FFI. Its hot path crosses two seams that this library implements for
 * real, and a Python host mirror (paper_2605_23945_b200) binds them with ctypes:
 *
 *   (1) the decode-step seam  oracle_decode_latency(hw, tp, B, T0 + B*arange(n))
 *       tpshift/latency.py:111-133, called at tpshift/engine.py:291-293; its
 *       HBM/compute terms (latency.py:123-124) are the projections below, its
 *       KV term is tps_paged_attention, its TP comm term (latency.py:125-126) is
 *       tps_reduce_push + the waiting tps_add_norm.
 *   (2) the switch seam       _commit_switch, tpshift/engine.py:206-269, and the
 *       plans it executes, plan_weight_reshard / plan_kv_migration
 *       (tpshift/reshard.py:80-151): tps_copy_items (weight pulls), tps_kv_move_items
 *       (plan_kv_migration's pages, expanded on the device), tps_barrier; the
 *       communication-group pool (tpshift/switchcost.py:76-104) is the IPC set.
 *
 * Device waits are bounded: a wait over its budget raises the soft-abort word
 * (tps_abort_status) and abandons instead of trapping.
 *
 * Conventions: every entry point takes raw device pointers, integer sizes and a
 * cudaStream_t passed as void*; calls are stream-ordered and asynchronous; the
 * library never allocates on the hot path (PyTorch owns every buffer). Return
 * value 0 = OK; TPS_EINVAL maps to tpshift ConfigError (tpshift/errors.py:8),
 * TPS_EPLAN to PlanVerificationError (tpshift/errors.py:36), TPS_ECUDA to a
 * RuntimeError carrying tps_last_error().
 *
 * bf16 tensors are passed as void*; fp32 as float*; all matrices row-major.
 */
#ifndef TPSHIFT_B200_H_
#define TPSHIFT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPS_OK 0
#define TPS_EINVAL (-22)
#define TPS_EPLAN (-1001)
#define TPS_ECUDA (-1002)

/* Completion-counter wait: spin until *ctr >= (*epoch) * mult + add
 * (epoch may be NULL -> target = add). NULL spec = no wait. */
typedef struct tps_wait {
  const uint64_t* ctr;
  const uint64_t* epoch;
  uint64_t mult;
  uint64_t add;
} tps_wait;

/* One contiguous chunk of a reshard / migration copy (32 bytes, device array). */
typedef struct tps_copy_item {
  const void* src;
  void* dst;
  uint64_t bytes;
  uint64_t reserved;
} tps_copy_item;

/* One KV migration move: a migrating sample x a run of n_heads kv heads that
 * are contiguous in the source and destination pools and pulled from one
 * source rank (tpshift/reshard.py:113-151, merge-first). Pools are
 * [L][2][num_pages][n_kv][64][D] bf16; page-table rows are int32. first_item =
 * exclusive prefix of L * 2 * n_pages over the moves array. */
typedef struct tps_kv_move {
  const void* src_kv;          /* source rank's pool base (local or IPC-mapped peer) */
  const int32_t* src_pages;    /* the sample's page-table row on the source rank */
  const int32_t* dst_pages;    /* the sample's page-table row on this rank */
  int32_t src_num_pages, src_nkv, src_head;
  int32_t dst_head, n_heads, n_pages;  /* n_pages = ceil(kv tokens / 64) */
  int64_t first_item;
} tps_kv_move;

/* ---------------------------------------------------------------- setup --- */
/* Soft watchdog: a device wait that exceeds its 20 s budget prints, raises this word
 * (nonzero code) and abandons its wait instead of trapping; every wait that has lasted
 * over 1 ms polls it and abandons too. Results computed after a raise are garbage: the
 * host must check the word (the Python binding does on every checked call) and fail. */
unsigned int tps_abort_status(void);
void tps_abort_clear(void);

/* Library/ABI version string. */
const char* tps_version(void);
/* Last error text of the calling thread (valid until the next failing call). */
const char* tps_last_error(void);
/* Bind the calling thread to `device`, report its SM count; checks sm_100 and
 * configures kernel attributes (call before any stream capture). */
int tps_init(int device, int* sm_count);
/* Programmatic dependent launch for decode-step kernels (default on). */
void tps_set_pdl(int on);

/* ------------------------------------------------ decode step (seam 1) --- */
/* Split-K count tps_linear will use for an [n x k] weight at batch b. */
int tps_linear_splits(int64_t n, int64_t k, int64_t b);

/* Column/row-parallel projection on tcgen05 tensor cores:
 *   out[s][i][j] = sum_{kk in split s} W[j][kk] * X[i][kk],  i < b, j < n
 * W: bf16 [n][ldw], X: bf16 [x_rows][ldx] (rows >= b are ignored), out: fp32
 * [splits][b][n]. Replaces the weight-traffic/compute term of
 * oracle_decode_latency (tpshift/latency.py:123-124). */
int tps_linear(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
               int64_t x_rows, int64_t ldx, float* out, int splits, void* stream);

/* Row-parallel projection with the TP allreduce fused into its epilogue (O and
 * down projections; the comm term of oracle_decode_latency, tpshift/latency.py:125-126):
 * every split-K partial tile is stored straight into each destination -- this
 * rank's slots in every TP peer's receive area, NVLink P2P stores -- at
 * dsts[d] + split * split_stride + i * n + j (fp32); the last CTA of the launch
 * then adds 1 to every sig_ctrs[] counter (release, system scope; `done` is the
 * launch site's CTA counter). The consumer (tps_add_norm with a counter wait)
 * sums the tp x splits slots in (rank, split) order. */
int tps_linear_push(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                    int64_t x_rows, int64_t ldx, float* const* dsts, int ndst, int64_t split_stride,
                    int splits, uint64_t* const* sig_ctrs, int nsig, unsigned int* done, void* stream);

/* LL form of tps_linear_push for tail batches: each partial element is one 8-byte
 * system-scope store {fp32 bits (low), tag (high)}, tag = (*epoch) * tag_mult + tag_add,
 * at dsts[d] + split * split_stride + i * n + j (uint64 units). No counters, fences or
 * signal: the consumer (tps_add_norm_ll) polls the tags (NCCL's LL protocol). */
int tps_linear_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                       int64_t x_rows, int64_t ldx, uint64_t* const* dsts, int ndst, int64_t split_stride,
                       int splits, const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add, void* stream);

/* resid[b] += sum of the nsrc LL slots (ll + i * stride, uint64 {value, tag}, polled until
 * every tag == (*epoch) * tag_mult + tag_add), then RMSNorm -> out (bf16). ctr (optional):
 * this phase's arrival counter, advanced by `bump` (= tp) so it stays at epoch * tp as if
 * the counter protocol had run (a layout's steps may use either protocol). */
int tps_add_norm_ll(float* resid, const uint64_t* ll, int nsrc, int64_t stride, const uint64_t* epoch,
                    uint32_t tag_mult, uint32_t tag_add, const void* w, float eps, int H, int B, void* out,
                    int ldo, uint64_t* ctr, uint64_t bump, void* stream);

/* Gate/up projection with the SwiGLU fused into the epilogue (no split-K):
 * W rows are 64-row blocks [gate c | up c] (n = 2F, F % 64 == 0);
 * act[i][f] = bf16(silu(gate_f . x_i) * (up_f . x_i)), act: bf16 [b][ld_act]. */
int tps_linear_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                    int64_t x_rows, int64_t ldx, void* act, int64_t ld_act, void* stream);

/* Row indirection used by every decode kernel: row b processes sample slot
 * row_slot[b] (< 0: padding row) at position row_pos[b], or at pos_by_slot[slot]
 * when row_pos is NULL (decode); row_pos lets one launch process several prompt
 * positions of a sample (chunked prefill through the decode kernels). */

/* resid[b] = E[history[slot][pos]] (replicated vocab table). */
int tps_embed(const int* row_slot, const int* pos_by_slot, const int* row_pos, const int* history,
              int hist_ld, const void* table, int H, int B, float* resid, void* stream);

/* Strided source convention (src, nsrc, src_stride): nsrc fp32 buffers at
 * src + i*src_stride (elements), summed in index order -- the split-K partials
 * of one projection, or one receive slot per TP rank (rank order). */

/* resid[b] += sum_i src_i[b], then out[b] = bf16(RMSNorm(resid[b]) * w); each
 * src_i is fp32 [B][H]. Consumer of the O/down projections and of the TP
 * allreduce receive slots; waits on `wait` first (NULL = no wait). */
int tps_add_norm(float* resid, const float* src, int nsrc, int64_t src_stride, const tps_wait* wait,
                 const void* w, float eps, int H, int B, void* out, int ldo, void* stream);

/* One-shot TP allreduce, push half (reference comm term, tpshift/latency.py:125-126):
 * r = sum_i srcs[i] (fp32, n elements), stored to every dsts[d] (this rank's slot
 * in each TP peer's receive area, NVLink P2P stores), then +1 on every sig_ctrs[]
 * (issued once per launch by the last CTA; `done` is that launch site's CTA counter). */
int tps_reduce_push(const float* src, int nsrc, int64_t src_stride, float* const* dsts, int ndst, int64_t n,
                    uint64_t* const* sig_ctrs, int nsig, unsigned int* done, void* stream);

/* LL form of tps_reduce_push: the summed [n] fp32 row block goes to every destination as
 * uint64 {value, tag} pairs (tag = (*epoch) * tag_mult + tag_add); no counters -- the
 * consumer is tps_add_norm_ll over the tp slots. */
int tps_reduce_push_ll(const float* src, int nsrc, int64_t src_stride, uint64_t* const* dsts, int ndst, int64_t n,
                       const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add, void* stream);

/* Split count of tps_linear_push_ll_cluster for [n x k] at batch b (0: not supported:
 * b > 64 or more tiles than SMs). */
int tps_cluster_splits(int64_t n, int64_t k, int64_t b);

/* LM head with greedy argmax stage 1 in the epilogue (split-K 1): logits [b][n] fp32 and, per
 * row i and 128-column tile t, cand[i * ceil(n/128) + t] = {max logit, smallest vocab index on
 * ties} (index = vocab0 + column) -- the candidates tps_argmax_finalize merges with
 * nchunk = ceil(n / 128); the same token tps_argmax_stage1 + finalize would pick. */
int tps_linear_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                      int64_t x_rows, int64_t ldx, float* logits, void* cand, int vocab0, void* stream);

/* Row-parallel projection + allreduce push with the split-K reduction inside the kernel:
 * the split CTAs of a weight tile form one cluster and sum their partials over DSMEM (split
 * order), then out[i][j] goes to every destination as ONE uint64 {fp32 bits, tag} at
 * dsts[d] + i * n + j (tag = (*epoch) * tag_mult + tag_add): the tp-source consumer is
 * tps_add_norm_ll, as after tps_reduce_push_ll. */
int tps_linear_push_ll_cluster(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                               int64_t x_rows, int64_t ldx, uint64_t* const* dsts, int ndst,
                               const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add, void* stream);

/* Tail-batch projections on CUDA cores (warp-shuffle GEMV, b <= tps_gemv_max_rows()): the
 * contracts of the tcgen05 family above at the tail, so the executor swaps one call for the
 * other (weight-traffic term of oracle_decode_latency, tpshift/latency.py:123-124):
 *   tps_gemv          = tps_linear with splits = 1: out fp32 [b][n]
 *   tps_gemv_silu     = tps_linear_silu (W rows in 64-row [gate c | up c] blocks, n = 2F)
 *   tps_gemv_push_ll  = tps_linear_push_ll_cluster: out[i][j] as one LL {fp32 bits, tag} at
 *                       dsts[d] + i * n + j, tag = (*epoch) * tag_mult + tag_add
 *   tps_gemv_argmax   = tps_linear_argmax: logits [b][n] + cand[i * ceil(n/128) + t]
 * k, ldw, ldx multiples of 8; w, x 16-byte aligned. Deterministic (fixed reduction order). */
int tps_gemv_max_rows(void);
int tps_gemv(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
             float* out, void* stream);
int tps_gemv_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                  void* act, int64_t ld_act, void* stream);
int tps_gemv_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                     uint64_t* const* dsts, int ndst, const uint64_t* epoch, uint32_t tag_mult, uint32_t tag_add,
                     void* stream);
int tps_gemv_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t ldx,
                    float* logits, void* cand, int vocab0, void* stream);

/* Positions per group of tps_prefill_attention for G query heads per KV head
 * (min(16, 64 / G); 0 if G > 64). */
int tps_prefill_group_positions(int G);

/* Chunked-prefill attention by sample group: group y (grid y < max_groups) is the
 * grp_n[y] rows grp_rows[y * 16 + i] of one sample (same row_slot; grp_n[y] <= 16 and
 * grp_n[y] * G <= 64; groups numbered densely: the first y with grp_n[y] == 0 ends the
 * table). One CTA per (group, KV head) streams the
 * sample's pages once for all its rows; row r attends to tokens 0..row_pos[r] (causal).
 * out: bf16 [rows][nq][D] for the grouped rows (others untouched). Same result as
 * tps_paged_attention with row_pos (prefill form) up to fp32 summation order. */
int tps_prefill_attention(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                          const int* row_pos, const int* grp_rows, const int* grp_n, int max_groups,
                          const int* page_table, int max_pages, int nq, int nkv, int D, void* out,
                          void* stream);

/* QKV: sum split partials [s][B][(nq+2nkv)*D] + bias, rotate-half RoPE (fp32
 * cos/sin tables [pos][D/2]), q -> bf16 [B][nq][D], k/v appended at each
 * row's position into the paged cache [page][nkv][64][D]. */
int tps_qkv_rope_append(const float* src, int nsrc, int64_t src_stride, const void* bias, const int* row_slot,
                        const int* pos_by_slot, const int* row_pos, const int* page_table, int max_pages,
                        const float* cos_t,
                        const float* sin_t, int B, int nq, int nkv, int D, int page_size, void* q_out,
                        void* k_cache, void* v_cache, void* stream);

/* Split policy for tps_paged_attention: -1 = one thread-block cluster per (row, kv head)
 * segment (tail batches, B x nkv <= 8); n = one wave of fixed splits when it fills >= 80 %
 * of the resident CTA slots; 0 = page-balanced schedule (more segments than slots, B <= 512). */
int tps_attn_splits(int B, int nkv, int max_pages);
/* fp32 elements of part_o a tps_paged_attention call needs (part_m / part_l: that / D);
 * nsplit = 0 selects the page-balanced schedule. */
int64_t tps_attn_workspace(int B, int nq, int D, int nsplit);

/* Paged GQA decode attention over ctx = pos+1 tokens per row, out bf16 [B][nq][D].
 * nsplit = 0 (default): page-balanced schedule -- the (row, kv head, page) units of
 * the launch are divided evenly over a persistent grid of resident CTAs, whatever the
 * context lengths; a (row, kv head) cut between CTAs is merged (log-sum-exp) by its
 * last piece. nsplit > 0: fixed split-KV per (row, kv head), merged by the last CTA.
 * nsplit = -1: a cluster of 8-16 CTAs per (row, kv head) splits the pages and merges the
 * softmax states through distributed shared memory (no scratch, no atomics).
 * part_m/part_l/part_o: fp32 scratch of tps_attn_workspace elements (part_o; the
 * others / D); merge_ctr: zero-initialised uint32 [B][nkv] (self re-arming). B <= 512
 * for the balanced form. KV term of tpshift/latency.py:123. */
int tps_paged_attention(const void* q, const void* k_cache, const void* v_cache, const int* row_slot,
                        const int* pos_by_slot, const int* row_pos, const int* page_table, int max_pages,
                        int B, int nq,
                        int nkv, int D, int nsplit, float* part_m, float* part_l, float* part_o,
                        unsigned int* merge_ctr, void* out, const float* qkv, int nqkv, int64_t qkv_stride,
                        const void* qkv_bias, const float* cos_t, const float* sin_t, void* stream);
/* Fused decode form (qkv != NULL, row_pos == NULL, nsplit > 0): q is not read; each CTA finishes its
 * KV group's queries from the QKV split partials (sum + bias + RoPE), and the CTA owning
 * the current token's page also appends that token's k/v to the cache -- the separate
 * tps_qkv_rope_append launch is not needed. */

/* act[b][f] = bf16(silu(g) * u) from split partials [s][B][2F] = [gate | up]. */
int tps_silu_mul(const float* src, int nsrc, int64_t src_stride, int B, int F, void* out, int ldo,
                 void* stream);

/* Vocab-parallel greedy argmax, stage 1: per-(row, chunk) (max, smallest global
 * index) candidates from LM-head split partials [s][B][V]; signals sig_ctrs. */
int tps_argmax_stage1(const float* src, int nsrc, int64_t src_stride, int B, int V, int vocab_offset,
                      int nchunk, void* cand, uint64_t* const* sig_ctrs, int nsig, unsigned int* done,
                      void* stream);

/* Stochastic form of tps_argmax_stage1 (the non-greedy sampler state of a sample is its
 * key seeds[row_slot[b]] and its position): candidates are the argmax over the rank's
 * vocab slice of logit / temperature + Gumbel(u), u from Philox4x32-10 with counter
 * (pos + 1, global vocab index, 0, 0) and the 64-bit key -- Gumbel-max, an exact draw
 * from softmax(logit / temperature), identical for any TP degree
 * (oracle/sampler_ref.py). pos = row_pos[b] when given, else pos_by_slot[slot]. */
int tps_sample_stage1(const float* src, int nsrc, int64_t src_stride, int B, int V, int vocab_offset, int nchunk,
                      void* cand, uint64_t* const* sig_ctrs, int nsig, unsigned int* done, const uint64_t* seeds,
                      const int* row_slot, const int* pos_by_slot, const int* row_pos, float temperature,
                      void* stream);

/* Stage 2: reduce candidates of all TP ranks (list = rank order), append the
 * token to history[slot][pos+1] unless pos+1 is still inside the prompt
 * (prompt_len may be NULL), advance pos_by_slot[slot]. out_tok may be NULL. */
int tps_argmax_finalize(const void* const* cands, int ncand, int nchunk, const tps_wait* wait, int B,
                        const int* row_slot, int* pos_by_slot, const int* prompt_len, int* history,
                        int hist_ld, int* out_tok, void* stream);

/* *epoch += 1 (end of a decode step; drives graph-replay-safe counter waits). */
int tps_epoch_advance(uint64_t* epoch, void* stream);

/* out[i] = sum_s src_s[i] for i < n (fp32). */
int tps_sum_partials(const float* src, int nsrc, int64_t src_stride, int64_t n, float* out, void* stream);

/* --------------------------------------------------- switch (seam 2) ----- */
/* Execute n copy items (device array of tps_copy_item). mode 0 = LSU vector
 * copy, 1 = TMA bulk (cp.async.bulk) staged copy. grid <= 0 -> 2 x SMs.
 * Replaces the All-Gather + Slice of tpshift/reshard.py:80-151. */
int tps_copy_items(const tps_copy_item* items, int n, int mode, int grid, void* stream);

/* Expand n_moves KV moves (device array) into n_items copy items (one per
 * (layer, k|v, valid page) of each move: n_heads x chunk_bytes contiguous in
 * both pools) written to items_out, ready for tps_copy_items. Page indices are
 * read from the page tables on the device, so the host plans O(samples)
 * descriptors. Out-of-range pages or head runs produce empty items and count
 * into *bad_pages (may be NULL). Replaces plan_kv_migration's per-chunk plan
 * (tpshift/reshard.py:113-151). */
int tps_kv_move_items(const tps_kv_move* moves, int n_moves, int64_t n_items, void* dst_kv, int dst_num_pages,
                      int dst_nkv, int64_t chunk_bytes, tps_copy_item* items_out, int* bad_pages, void* stream);

/* Device barrier over the node's ranks (the switch's two barriers, tpshift/engine.py:
 * 206-269): store `epoch` (monotone, one per barrier) into this rank's slot of every
 * peer's slot array (peer_slots[i] = &peer_i_slots[self_slot]), then wait until
 * my_slots[j] >= epoch for every j != self_slot, j < nslots. One slot per source, so a
 * rank already at the next barrier cannot release a slower rank early. */
int tps_barrier(uint64_t* const* peer_slots, int npeers, const uint64_t* my_slots, int nslots, int self_slot,
                uint64_t epoch, void* stream);

/* CUDA IPC for the Cache Manager's per-(tp, dp) peer tables
 * (CommGroupPool, tpshift/switchcost.py:76-104). handle: 64 bytes. */
int tps_ipc_get_handle(const void* ptr, void* handle_out, int64_t* offset_out);
int tps_ipc_open(const void* handle, void** base_out);
int tps_ipc_close(void* base);

/* Device step tracer (probe): while registered, thread 0 of block 0 of every decode
 * kernel appends a record [kind, t_entry, t_after_wait, t_exit] (uint64, %globaltimer ns)
 * at records[4 * atomicAdd(counter, 1)] (up to `capacity` records). NULL, NULL disables. */
int tps_trace_enable(uint64_t* records, unsigned int* counter, unsigned int capacity);


/* ------------------------------------------------ persistent decode step --- *
 * One launch per decode step for tail batches (B <= 16, head_dim 128): the whole step
 * (embedding, every layer's QKV / RoPE + paged KV append / attention / O + TP allreduce /
 * RMSNorm / gate-up + SiLU / down + TP allreduce, LM head, greedy argmax) in one cooperative
 * grid of one CTA per SM per rank. Replaces, for the post-switch tail, the same
 * oracle_decode_latency step (tpshift/latency.py:111-133) the per-kernel entry points above
 * implement; the TP allreduce uses the LL slots of tps_linear_push_ll (S = 1 layout) and the
 * phase counters stay at epoch * tp, so a layout may alternate between the two forms. */
typedef struct tps_persist_geom {
  int num_layers;
  int hidden;
  int head_dim;   /* 128 */
  int n_phases;   /* 2 * num_layers + 1 (LL tag = epoch * n_phases + phase) */
  float rms_eps;
} tps_persist_geom;

typedef struct tps_persist_rank {
  /* weights: arrays of num_layers device pointers (bf16, row-major, the rank's shard) */
  const void* const* w_qkv;
  const void* const* b_qkv;       /* NULL array: no bias */
  const void* const* w_o;
  const void* const* w_gu;        /* interleaved 64-row [gate | up] blocks */
  const void* const* w_d;
  const void* const* ln1;
  const void* const* ln2;
  const void* embed;
  const void* ln_f;
  const void* lm_head;
  void* const* k_cache;           /* per layer [pages][nkv][64][128] */
  void* const* v_cache;
  int nq, nkv, ffn, vocab, vocab_off;  /* local query / KV heads, FFN width, vocab rows, offset */
  int nq_of[8];                   /* query heads of every rank of the group (rank order) */
  /* slot state (tps_paged_attention / tps_argmax_finalize conventions) */
  const int* row_slot;
  int* pos;
  const int* page_table;
  int max_pages;
  int* history;
  int hist_ld;
  const int* prompt_len;
  int* out_tok;
  float* logits;                  /* [16][vocab] fp32 logits of the step (parity checks) */
  const float* cos_t;             /* [max_pos][64] */
  const float* sin_t;
  void* work;                     /* zero-initialised, tps_persist_work_bytes() bytes */
  int64_t work_bytes;
  /* TP exchange (tp > 1): LL areas [2][src][rows][hidden] uint64 and argmax areas
   * [2][8][16][2] uint64 of every rank (rank order); loopback: this rank plays every peer */
  int tp, rank, loopback;
  int64_t ll_par_stride, ll_src_stride;
  uint64_t* ll_peer[8];
  uint64_t* ll_mine;
  uint64_t* am_peer[8];
  uint64_t* am_mine;
  uint64_t* epoch;                /* group epoch (advanced by the step) */
  uint64_t* ctr;                  /* group phase counters (kept at epoch * tp) */
  uint64_t* trace;                /* probe (or NULL): [CTA][16] %globaltimer marks of layer trace_layer */
  int trace_layer;
} tps_persist_rank;

/* sizeof(tps_persist_geom) (which 0) / sizeof(tps_persist_rank) (which 1): binding check. */
int64_t tps_persist_struct_bytes(int which);
/* 1 if the persistent step supports this rank's shapes at batch B. */
int tps_persist_supported(const tps_persist_geom* g, const tps_persist_rank* r, int B);
/* Bytes of the per-rank workspace (counters, residual, partials, logits) for `ctas` CTAs. */
int64_t tps_persist_work_bytes(const tps_persist_geom* g, const tps_persist_rank* r, int ctas);
/* Bytes of a launch context for nranks ranks. */
int64_t tps_persist_ctx_bytes(const tps_persist_geom* g, int nranks);
/* Encode the tensor maps and pointer tables of nranks ranks (one process's ranks of one
 * group: the whole virtual group, or a single rank) for bucket B into dev_ctx (synchronous). */
int tps_persist_prepare(const tps_persist_geom* g, const tps_persist_rank* ranks, int nranks, int B, int ctas,
                        void* dev_ctx, void* stream);
/* One decode step: nranks * ctas CTAs (cooperative), stream-ordered. */
int tps_persist_launch(const void* dev_ctx, int nranks, int ctas, int B, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TPSHIFT_B200_H_ */
