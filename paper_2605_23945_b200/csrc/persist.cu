// Persistent decode step for tail batches (B <= 16, head_dim 128): ONE launch per decode step.
//
// Replaces the ~9 launches per layer of the multi-kernel step (embed, add+norm, QKV GEMM,
// RoPE/append, attention, O GEMM + LL push, add+norm, gate/up GEMM, down GEMM + LL push, LM
// head, argmax) for the post-switch tail, where every launch boundary cost ~1.8 us against a
// per-layer weight stream of ~9 us (TP8 Qwen2.5-7B). The step being replaced is tpshift's
// oracle_decode_latency (tpshift/latency.py:111-133): the HBM term of its max(...) is the
// weight stream this kernel keeps busy, its comm term (latency.py:125-126) the LL exchange.
//
// Structure (one CTA per SM, cooperative launch, 8 consumer warps + 1 producer warp):
//
// * Weight stream. Every projection is cut into 16-row units; a unit streams as stages of
//   16 rows x 256 columns (8 KB, four 2-D TMA boxes, SWIZZLE_128B) into a 12-slot smem ring.
//   The producer warp walks the whole step's schedule (per layer QKV, O, gate/up, down; the
//   LM head) and never waits on data, only on ring slots, so weights keep streaming through
//   every dependency wait (norm, attention, the NVLink exchange) up to the ring's 96 KB.
// * Column-parallel projections (QKV, gate/up, LM head): each unit is complete output rows
//   over the full K, so its owner finishes it in registers -- no cross-CTA partials. QKV and
//   gate/up units pair 8 rows with the 8 rows 64 below them (the two halves of a rotary pair;
//   a gate row and its up row in the interleaved [gate | up] blocks): RoPE and SiLU(gate)*up
//   happen on the rows the unit just produced.
// * Row-parallel projections (O, down): "stream-K" -- the units' stages are dealt to the CTAs
//   as equal contiguous ranges, so a unit is split between at most two CTAs; each piece pushes
//   its partial straight into every TP peer's receive slot as LL {value, tag} pairs (slot =
//   rank * 2 + piece): the allreduce is fused into the projection epilogue over NVLink.
// * GEMV on the tensor pipe: the 8 warps split each stage's K (32 columns each), mma.sync
//   m16n8k16 with the weights as A (ldmatrix from the swizzled boxes) and the <= 16 rows of
//   activations as B from a padded smem window, reduced across warps per unit. At B <= 16 the
//   flops are ~1/100 of the pipe: HBM is the bound.
// * Residual + RMSNorm in slices: the owner CTA of each 128-column slice polls the peers' LL
//   slots, adds them to the fp32 residual in (rank, piece) order and publishes the slice's
//   sum of squares; consumers of the normed vector combine the slice sums in fixed order and
//   normalise their activation window on load -- the normed activation never goes to HBM.
// * Attention: units = (row, KV head, KV split); each streams its pages through the mma.sync
//   page kernel of the split decode attention; the last split of a (row, head) merges.
// * Dependencies: monotone progress counters (one arrival per CTA per phase; targets are a
//   function of the step, so CUDA-graph replays need no reset) and the LL tags; every wait
//   is watchdog-bounded.
//
// Numerics: bf16 storage exactly where the multi-kernel step stores bf16 (normed
// activations, q, K/V, attention output, SiLU*up), fp32 accumulation.
#include <algorithm>
#include <cstddef>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "attention_common.cuh"
#include "../../include/tpshift_b200.h"

namespace tps {


namespace pst {

constexpr int kUR = 16;                          // rows per unit
// A ring slot holds one 32 KB TMA box (3-D tensor map [chunk][row][64], SWIZZLE_128B): 16 rows x
// 1024 columns, or 8 rows x 2048 columns. Measured (tools/cuda/tma_stream_bench.cu, 148 CTAs):
// 32 KB boxes stream at 6.6-7.0 TB/s, 16 KB at 5.8, 2 KB (16 x 64) at 1.4 -- the TMA cost is
// per box, so small units need many-column boxes.
constexpr int kSlotBytes = 32 * 1024;
constexpr int kStages = 4;                       // ring slots (128 KB)
constexpr int kSKu = 1024;                       // columns per stage, unpaired (one 16-row box)
constexpr int kSKp = 2048;                       // columns per stage, paired (two 8-row boxes)
// 7 consumer warps + 1 producer warp: 8 warps = 2 per SM sub-partition, so a thread may hold
// 255 registers (9 warps would cap it at 168 and spill the attention accumulators)
constexpr int kCW = 7;                           // consumer warps
constexpr int kCT = kCW * 32;
constexpr int kThreads = kCT + 32;               // + producer warp
constexpr int kMaxB = 16;
constexpr int kWinBytes = 86 * 1024;             // activation window
constexpr int kRedBytes = 8 * kUR * kMaxB * 4;   // cross-warp reduction (<= 8 warps)
constexpr int kOutBytes = kUR * kMaxB * 4;       // one unit's result [16 rows][16 cols]
constexpr int kScratch = kWinBytes + kRedBytes + kOutBytes;
constexpr int kMisc = 2048;
constexpr int kSmem = kStages * kSlotBytes + kScratch + kMisc + 1024;  // + alignment slack
constexpr int kMaxSplit = 32;
constexpr int kMaxTP = 8;
enum Kind { kQKV = 0, kO = 1, kGU = 2, kDown = 3, kLM = 4 };

struct Geo {
  int L, H, B, C, nranks, n_phases, S_att, NS, max_units;
  float eps, scale_log2;
};

struct RankDev {
  const CUtensorMap* tmaps;                 // [4L + 1]: per layer qkv, o, gu, d; then lm_head
  const __nv_bfloat16* const* b_qkv;        // [L] (entries may be null)
  const __nv_bfloat16* const* ln1;          // [L]
  const __nv_bfloat16* const* ln2;          // [L]
  __nv_bfloat16* const* kc;                 // [L] layer bases [pages][nkv][64][128]
  __nv_bfloat16* const* vc;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* ln_f;
  int nq, nkv, F, V, voff;
  int nq_of[kMaxTP];                        // every rank's query heads (its O projection's K / 128)
  const int* row_slot;
  int* pos;
  const int* page_table;
  int max_pages;
  int* hist;
  int hist_ld;
  const int* prompt_len;
  int* out_tok;
  float* logits;                            // [16][V]
  const float* cos_t;
  const float* sin_t;
  // workspace (tps_persist_work_bytes)
  unsigned long long* prog;  // [0] step, [1] exit, [2] lm, [3..] norm[2L+1], qkv[L], att[L], act[L]
  unsigned int* att_cnt;     // [16 * nkv]
  float* resid;              // [16][H]
  __nv_bfloat16* q;          // [16][nq][128]
  __nv_bfloat16* attn;       // [16][nq * 128]
  __nv_bfloat16* act;        // [16][F]
  float* att_o;              // [max_units][16][128]
  float* att_m;              // [max_units][16]
  float* att_l;
  float* sq[2];              // [NS][16]
  ArgmaxCand* cand;          // [V / 16][16]
  // TP exchange (LL {value, tag}); tp == 1: a local area, tags from the step counter
  int tp, rank, loopback;
  long long ll_par_stride, ll_src_stride;   // elements
  uint64_t* ll_peer[kMaxTP];
  uint64_t* ll_mine;
  uint64_t* am_peer[kMaxTP];                // argmax candidates [2][8][16][2]
  uint64_t* am_mine;
  const uint64_t* ep;                       // LL tag epoch
  uint64_t* ep_adv;                         // advanced at step end (null: prog[0] is the epoch)
  unsigned long long* ctr;                  // group phase counters kept at epoch * tp (or null)
  unsigned long long* trace;                // probe: [CTA][16] %globaltimer marks of one layer (or null)
  int trace_layer;
};

struct Ctx {  // device-resident launch context: Geo then RankDev[nranks]
  Geo g;
  RankDev r[1];
};

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(kCT) : "memory"); }

__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin with relaxed loads (an acquire load per poll would invalidate L1 every iteration), then
// one acquire fence once the target is reached.
__device__ __forceinline__ void wait_geq(const unsigned long long* p, unsigned long long target, int what) {
  if (ld_rlx(p) < target) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_rlx(p) < target) {
      bool fired = false;
      if (wait_abandoned(t0, &fired)) {
        if (fired) {
          printf("tps persist watchdog: wait %d block %d at %llu < %llu\n", what, blockIdx.x, ld_rlx(p), target);
          raise_abort(4);
        }
        break;
      }
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// consumer-wide wait on a progress counter (thread 0 spins, the others meet it at the barrier)
__device__ __forceinline__ void cwait(const unsigned long long* p, unsigned long long target, int what) {
  if (threadIdx.x == 0) wait_geq(p, target, what);
  cbar();
}

// acquire-release fence at gpu scope (one thread; the CTA's other threads are ordered through a
// barrier). __threadfence() is a sequentially consistent fence and costs far more under load.
__device__ __forceinline__ void fence_ar() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// one arrival (release: the CTA's stores, ordered before by the preceding barrier, are visible first)
__device__ __forceinline__ void signal(unsigned long long* p) {
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

// ------------------------------------------------------------ schedule ---
struct Phase {
  int kind, N, K, U, ns, sk;  // rows, columns, 16-row units, stages per unit, columns per stage
  bool paired;            // unit = 8 rows + the 8 rows 64 below (QKV, gate/up)
  bool row_par;           // stream-K split over CTAs (O, down)
};

__device__ __forceinline__ Phase phase_of(const RankDev& R, const Geo& g, int kind, int nq) {
  Phase p;
  p.kind = kind;
  switch (kind) {
    case kQKV: p.N = (nq + 2 * R.nkv) * 128; p.K = g.H; break;
    case kO: p.N = g.H; p.K = nq * 128; break;
    case kGU: p.N = 2 * R.F; p.K = g.H; break;
    case kDown: p.N = g.H; p.K = R.F; break;
    default: p.N = R.V; p.K = g.H; break;
  }
  p.U = (p.N + kUR - 1) / kUR;
  p.paired = kind == kQKV || kind == kGU;
  p.sk = p.paired ? kSKp : kSKu;
  p.ns = (p.K + p.sk - 1) / p.sk;
  p.row_par = kind == kO || kind == kDown;
  return p;
}

// [lo, hi) of an n-item list dealt over C CTAs (balanced, contiguous)
__device__ __forceinline__ int span_lo(int c, int n, int C) { return (int)(((long long)c * n + C - 1) / C); }
// stream-K ranges of a row-parallel phase: CTAs [0, Ce) hold T = U * ns stages
__device__ __forceinline__ int row_ctas(const Phase& p, const Geo& g) { return min(g.C, p.U); }
__device__ __forceinline__ long long rng_lo(int c, long long T, int Ce) { return (long long)c * T / Ce; }
__device__ __forceinline__ int rng_owner(long long x, long long T, int Ce) { return (int)(((x + 1) * Ce - 1) / T); }
// a unit of a row-parallel phase is split between two CTAs?
__device__ __forceinline__ bool unit_split(int u, int ns, int U, int Ce) {
  const long long T = (long long)U * ns;
  return rng_owner((long long)u * ns, T, Ce) != rng_owner((long long)u * ns + ns - 1, T, Ce);
}

// ------------------------------------------------------------------ producer ---
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

// Stage st of unit u: one box (unpaired: rows u*16.., 16 chunks of 64 columns) or two (paired:
// 8 rows and the 8 rows 64 below, 32 chunks each), one ring slot per box. Boxes past K are
// zero-filled by the TMA unit (full box bytes are still delivered).
__device__ void producer(const RankDev& R, const Geo& g, int c, uint8_t* ring, uint64_t* full, uint64_t* empty) {
  const uint64_t pol = policy_evict_first();
  uint32_t it = 0;
  const int nph = 4 * g.L + 1;
  auto slot_for = [&](void) -> uint32_t {
    const uint32_t slot = it % kStages;
    if (it >= kStages) mbar_wait(&empty[slot], ((it / kStages) + 1) & 1);
    mbar_arrive_expect_tx(&full[slot], kSlotBytes);
    return slot;
  };
  for (int ph = 0; ph < nph; ++ph) {
    const int kind = ph == 4 * g.L ? kLM : (ph & 3);
    const Phase p = phase_of(R, g, kind, R.nq);
    const CUtensorMap* tm = R.tmaps + ph;
    auto next = [&](int u, int st) {
      if (R.trace != nullptr && kind == kQKV && ph / 4 == R.trace_layer) {  // probe: issue times
        const uint64_t t = globaltimer_ns();
        if (R.trace[c * 32 + 31] < ((unsigned long long)g.L << 40)) R.trace[c * 32 + 31] = t;  // (first)
        R.trace[c * 32 + 15] = t;  // last
      }
      const int chunk = st * (p.sk / 64);
      if (p.paired) {
        const int row0 = (u >> 3) * 128 + (u & 7) * 8;
        uint32_t slot = slot_for();
        tma_load_3d(ring + slot * kSlotBytes, tm, &full[slot], 0, row0, chunk, pol);
        ++it;
        slot = slot_for();
        tma_load_3d(ring + slot * kSlotBytes, tm, &full[slot], 0, row0 + 64, chunk, pol);
        ++it;
      } else {
        const uint32_t slot = slot_for();
        tma_load_3d(ring + slot * kSlotBytes, tm, &full[slot], 0, u * kUR, chunk, pol);
        ++it;
      }
    };
    if (p.row_par) {
      const int Ce = row_ctas(p, g);
      if (c >= Ce) continue;
      const long long T = (long long)p.U * p.ns;
      for (long long x = rng_lo(c, T, Ce); x < rng_lo(c + 1, T, Ce); ++x) next((int)(x / p.ns), (int)(x % p.ns));
    } else {
      for (int u = span_lo(c, p.U, g.C); u < span_lo(c + 1, p.U, g.C); ++u)
        for (int st = 0; st < p.ns; ++st) next(u, st);
    }
  }
}

// -------------------------------------------------------------- smem layout ---
struct Smem {
  uint8_t* ring;
  uint8_t* scratch;   // window | reduction | unit result (also: attention stages, norm sources)
  float* red;         // [8 warps][16 cols][16 rows]
  float* out;         // [16 cols (batch rows)][16 unit rows]
  uint64_t* full;
  uint64_t* empty;
  float* rstd;        // [16]
  int* flag;          // [4]
  int* rslot;         // [16] row -> slot (-1: padding row)
  int* rpos;          // [16] position processed this step
  int* rpage;         // [16] page holding that position
  int* rtok;          // [16] token at that position
  int* rsa;           // [16] attention splits of the row
  int* rub;           // [17] first attention unit of the row (prefix sum; rub[B] = units)
  float* wred;        // [16] small reductions
  float* lmv;         // [16] LM head: running best value of the row over this CTA's units
  int* lmi;           // [16] ... and its index
};

__device__ __forceinline__ void trace_ev(const RankDev& R, int c, int l, int ev) {
  if (R.trace != nullptr && l == R.trace_layer && threadIdx.x == 0) R.trace[c * 32 + ev] = globaltimer_ns();
}

// ------------------------------------------------------- activation window ---
// The B (<= 16) activation rows of k columns [k0, k1) as bf16 in smem, padded rows (B
// fragments conflict-free). mode 0: xn = bf16(resid * rstd * w) (RMSNorm on load); mode 1:
// bf16 copy of src [B][ld]. Loads are issued in batches of 4 per thread.
struct Window {
  int k0, k1, ld;  // resident columns and row pitch (elements)
  int tr = -1, l = 0;           // probe: CTA index / layer of a traced window load
  const RankDev* R = nullptr;
};

// columns of B rows that fit the window (a multiple of 2048, i.e. of any stage)
__device__ __forceinline__ int win_rows(int B) { return B <= 8 ? 8 : 16; }
__device__ __forceinline__ int win_cap(int B) { return ((kWinBytes / (win_rows(B) * 2)) - 8) / kSKp * kSKp; }

// Rows [B, 8 * NT) are zero (the MMA's padding columns); only the B real rows are loaded. Row
// pitch cap + 8 elements: conflict-free B fragments.
__device__ void load_window(const Smem& S, Window& W, int mode, const float* resid, const __nv_bfloat16* w,
                            const __nv_bfloat16* src, int ld, int B, int k0, int k1) {
  __nv_bfloat16* xw = reinterpret_cast<__nv_bfloat16*>(S.scratch);
  const int tid = threadIdx.x;
  const int xld = win_cap(B) + 8;
  cbar();  // every warp is done with the previous window
  const int n = k1 - k0;  // multiple of 64
  for (int e = tid; e < (win_rows(B) - B) * (n / 8); e += kCT) {  // zero padding rows
    const int b = B + e / (n / 8), k = (e % (n / 8)) * 8;
    *reinterpret_cast<uint4*>(xw + b * xld + k) = make_uint4(0u, 0u, 0u, 0u);
  }
  if (mode == 0) {
    const int n4 = n / 4, tot = B * n4;
    for (int e0 = tid; e0 < tot; e0 += 4 * kCT) {
      float4 x[4];
      uint2 wv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = e0 + j * kCT;
        const int b = e / n4, k = (e - b * n4) * 4;
        if (e < tot) {
          x[j] = __ldcg(reinterpret_cast<const float4*>(resid + (size_t)b * ld + k0 + k));
          wv[j] = *reinterpret_cast<const uint2*>(w + k0 + k);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = e0 + j * kCT;
        if (e < tot) {
          const int b = e / n4, k = (e - b * n4) * 4;
          const float r = S.rstd[b];
          const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[j].x));
          const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[j].y));
          uint2 o;
          o.x = pack_bf16(x[j].x * r * a.x, x[j].y * r * a.y);
          o.y = pack_bf16(x[j].z * r * c.x, x[j].w * r * c.y);
          *reinterpret_cast<uint2*>(xw + b * xld + k) = o;
        }
      }
    }
  } else {
    const int n8 = n / 8, tot = B * n8;
    for (int e0 = tid; e0 < tot; e0 += 4 * kCT) {
      uint4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = e0 + j * kCT;
        const int b = e / n8, k = (e - b * n8) * 8;
        if (e < tot) v[j] = __ldcg(reinterpret_cast<const uint4*>(src + (size_t)b * ld + k0 + k));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = e0 + j * kCT;
        if (e < tot) {
          const int b = e / n8, k = (e - b * n8) * 8;
          *reinterpret_cast<uint4*>(xw + b * xld + k) = v[j];
        }
      }
    }
  }
  cbar();
  W.k0 = k0;
  W.k1 = k1;
  W.ld = xld;
  if (W.tr >= 0) trace_ev(*W.R, W.tr, W.l, 30);
}

// ----------------------------------------------------------------- unit MMA ---
// Stream stages [st0, st1) of unit u through the ring into the warp's accumulators: warp w
// takes every 8th 16-column step of a stage. A slot holds [chunk][rows][64] (128-byte rows,
// 16-byte pieces XOR-swizzled by row & 7); paired stages take two slots (rows 0-7 | 8-15).
// kAcc independent accumulator sets per warp: consecutive k-steps of a warp do not wait on
// each other's HMMA (the legacy mma.sync pipe has a long dependent-issue latency)
constexpr int kAcc = 4;

// Per-thread accumulators of a unit: the tensor-pipe form (NT n-tiles of 8 batch rows, kAcc
// sets) or, FB > 0, the CUDA-core form (FB batch rows of one weight row).
template <int NT, int FB>
struct Acc {
  float m[kAcc][NT][4];
  float f[FB > 0 ? FB : 1];
};

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ float dot8(uint4 w, uint4 x, float acc) {
  const uint32_t wa[4] = {w.x, w.y, w.z, w.w}, xa[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 wf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wa[i]));
    const float2 xf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xa[i]));
    acc = fmaf(wf.x, xf.x, acc);
    acc = fmaf(wf.y, xf.y, acc);
  }
  return acc;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Tail batches (FB = B <= 4) use CUDA-core FMAs instead: thread (weight row tid % 16, column
// group tid / 16) reads 8 weights (one 16-byte swizzled piece) and the FB activation rows per
// step -- at B = 1 the m16n8k16 tensor form wastes 7/8 of every MMA and its issue rate, not
// HBM, bounded a stage.
template <int NT, int FB>
__device__ __forceinline__ void mma_stages(const Smem& S, Window& W, const Phase& p, int st0, int st1, uint32_t& it,
                                           Acc<NT, FB>& acc, int mode, const float* resid,
                                           const __nv_bfloat16* w, const __nv_bfloat16* src, int ld, int B) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, cq = lane & 3;
  const uint32_t ring0 = smem_u32(S.ring);
  const uint32_t xw0 = smem_u32(S.scratch);
  const int lrow = ((lane >> 3) & 1) * 8 + (lane & 7);  // ldmatrix: matrix m = lane / 8
  const int lhalf = lane >> 4;
  const int nslot = p.paired ? 2 : 1;
  const int csb = p.paired ? 8 * 128 : kUR * 128;     // bytes per 64-column chunk in a slot
  const uint32_t lsw = (uint32_t)(lrow & 7);
  const uint32_t lrowb = (uint32_t)((nslot == 2 ? (lrow & 7) : lrow) * 128);
  for (int st = st0; st < st1; ++st) {
    const int k0 = st * p.sk;
    const int kv = min(p.sk, p.K - k0);
    if (k0 < W.k0 || k0 + kv > W.k1)
      load_window(S, W, mode, resid, w, src, ld, B, k0, min(p.K, k0 + win_cap(B)));
    const uint32_t s0 = it % kStages, s1 = (it + 1) % kStages;
    mbar_wait(&S.full[s0], (it / kStages) & 1);
    if (nslot == 2) mbar_wait(&S.full[s1], ((it + 1) / kStages) & 1);
    // this lane's ldmatrix row (paired rows 8..15 live in the second slot) and B-fragment row
    const uint32_t rbase = ring0 + (nslot == 2 && lrow >= 8 ? s1 : s0) * kSlotBytes + lrowb;
    if constexpr (FB > 0) {
      constexpr int kGroups = kCT / 16;
      const int r = tid & 15, kg = tid >> 4;
      const int rr = nslot == 2 ? (r & 7) : r;
      const uint32_t wb = ring0 + (nslot == 2 && r >= 8 ? s1 : s0) * kSlotBytes + (uint32_t)(rr * 128);
      const uint32_t xb = xw0 + (uint32_t)((k0 - W.k0) * 2);
      const uint32_t sw = (uint32_t)(rr & 7);
      const int nc8 = kv / 8;
      for (int kc = kg; kc < nc8; kc += kGroups) {
        const uint4 wv = lds128(wb + (uint32_t)((kc >> 3) * csb) + (((uint32_t)(kc & 7) ^ sw) << 4));
#pragma unroll
        for (int b = 0; b < FB; ++b)
          acc.f[b] = dot8(wv, lds128(xb + (uint32_t)((b * W.ld + kc * 8) * 2)), acc.f[b]);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.empty[s0]);
        if (nslot == 2) mbar_arrive(&S.empty[s1]);
      }
      it += nslot;
      continue;
    }
    const uint32_t xb = xw0 + (uint32_t)((gq * W.ld + (k0 - W.k0) + 2 * cq) * 2);
    const uint32_t xnt = (uint32_t)(8 * W.ld * 2);
    const int nks = (kv + 15) / 16;
    for (int ks0 = warp; ks0 < nks; ks0 += kAcc * kCW) {
#pragma unroll
      for (int q = 0; q < kAcc; ++q) {
        const int ks = ks0 + q * kCW;
        if (ks < nks) {
          uint32_t a[4];
          const uint32_t j = (uint32_t)(((ks & 3) << 1) + lhalf);
          ldmatrix_x4(a, rbase + (uint32_t)((ks >> 2) * csb) + ((j ^ lsw) << 4));
          const uint32_t xk = xb + (uint32_t)(ks * 32);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            mma16816(acc.m[q][nt], a, lds32(xk + nt * xnt), lds32(xk + nt * xnt + 16));
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&S.empty[s0]);
      if (nslot == 2) mbar_arrive(&S.empty[s1]);
    }
    it += nslot;
  }
}

// Sum the 8 warps' accumulators (fixed order) -> S.out[b][r] (16 unit rows per batch row).
template <int NT, int FB>
__device__ __forceinline__ void reduce_unit(const Smem& S, Acc<NT, FB>& acc, int B) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if constexpr (FB > 0) {
    constexpr int kGroups = kCT / 16;
    const int r = tid & 15, kg = tid >> 4;
#pragma unroll
    for (int b = 0; b < FB; ++b) {
      S.red[(kg * FB + b) * kUR + r] = acc.f[b];
      acc.f[b] = 0.f;
    }
    cbar();
    for (int e = tid; e < B * kUR; e += kCT) {
      const int b = e >> 4, r2 = e & 15;
      float v = 0.f;
#pragma unroll
      for (int k = 0; k < kGroups; ++k) v += S.red[(k * FB + b) * kUR + r2];
      S.out[e] = v;
    }
    cbar();
    return;
  }
  const int gq = lane >> 2, cq = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = gq + ((e & 2) ? 8 : 0), col = nt * 8 + 2 * cq + (e & 1);
      float v = 0.f;
#pragma unroll
      for (int q = 0; q < kAcc; ++q) {
        v += acc.m[q][nt][e];
        acc.m[q][nt][e] = 0.f;
      }
      S.red[(warp * kMaxB + col) * kUR + row] = v;
    }
  cbar();
  for (int e = tid; e < B * kUR; e += kCT) {
    float v = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < kCW; ++w2) v += S.red[w2 * kMaxB * kUR + e];
    S.out[e] = v;
  }
  cbar();
}

// ------------------------------------------------------ column-parallel ---
// QKV / gate-up / LM head: units dealt to CTAs as contiguous spans, each finished in place.
// One arrival per CTA on `done` after its last unit (lm: the last CTA runs the argmax).
template <int NT, int FB>
__device__ void col_phase(const RankDev& R, const Geo& g, const Smem& S, int c, int l, int kind, uint32_t& it,
                          const float* resid, const __nv_bfloat16* w, unsigned long long* done,
                          unsigned long long e1, bool& final_lm) {
  const Phase p = phase_of(R, g, kind, R.nq);
  const int u0 = span_lo(c, p.U, g.C), u1 = span_lo(c + 1, p.U, g.C);
  const int tid = threadIdx.x, B = g.B;
  Window W{1 << 30, -1, 0};
  if (kind == kQKV) {
    W.tr = c;
    W.l = l;
    W.R = &R;
  }
  Acc<NT, FB> acc;
#pragma unroll
  for (int q = 0; q < kAcc; ++q)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc.m[q][nt][0] = acc.m[q][nt][1] = acc.m[q][nt][2] = acc.m[q][nt][3] = 0.f;
#pragma unroll
  for (int b = 0; b < (FB > 0 ? FB : 1); ++b) acc.f[b] = 0.f;
  const bool tr = kind == kQKV && u0 < u1;
  for (int u = u0; u < u1; ++u) {
    if (tr && u == u0) trace_ev(R, c, l, 26);
    mma_stages<NT, FB>(S, W, p, 0, p.ns, it, acc, 0, resid, w, nullptr, g.H, B);
    if (tr && u == u0) trace_ev(R, c, l, 27);
    reduce_unit<NT, FB>(S, acc, B);
    if (tr && u == u0) trace_ev(R, c, l, 28);
    const float* out = S.out;
    if (kind == kQKV) {
      const int h = u >> 3, j = u & 7;
      const __nv_bfloat16* bias = R.b_qkv[l];
      for (int e = tid; e < B * 8; e += kCT) {
        const int b = e >> 3, r = e & 7, i = 8 * j + r;
        float x0 = out[b * kUR + r], x1 = out[b * kUR + r + 8];
        if (bias) {
          x0 += bf2f(bias[h * 128 + i]);
          x1 += bf2f(bias[h * 128 + i + 64]);
        }
        const int slot = S.rslot[b], pos = S.rpos[b];
        if (h < R.nq) {
          __nv_bfloat16* q = R.q + ((size_t)b * R.nq + h) * 128;
          const float cs = R.cos_t[(size_t)pos * 64 + i], sn = R.sin_t[(size_t)pos * 64 + i];
          q[i] = f2bf(x0 * cs - x1 * sn);
          q[i + 64] = f2bf(x1 * cs + x0 * sn);
        } else if (slot >= 0) {
          const bool isk = h < R.nq + R.nkv;
          const int jh = isk ? h - R.nq : h - R.nq - R.nkv;
          const size_t off = (((size_t)S.rpage[b] * R.nkv + jh) * kPage + (pos % kPage)) * 128;
          if (isk) {
            const float cs = R.cos_t[(size_t)pos * 64 + i], sn = R.sin_t[(size_t)pos * 64 + i];
            R.kc[l][off + i] = f2bf(x0 * cs - x1 * sn);
            R.kc[l][off + i + 64] = f2bf(x1 * cs + x0 * sn);
          } else {
            R.vc[l][off + i] = f2bf(x0);
            R.vc[l][off + i + 64] = f2bf(x1);
          }
        }
      }
    } else if (kind == kGU) {
      const int f0 = (u >> 3) * 64 + (u & 7) * 8;
      for (int e = tid; e < B * 8; e += kCT) {
        const int b = e >> 3, r = e & 7;
        const float gt = out[b * kUR + r], up = out[b * kUR + r + 8];
        R.act[(size_t)b * R.F + f0 + r] = f2bf(gt / (1.f + __expf(-gt)) * up);
      }
    } else {  // LM head: fp32 logits + the running per-row candidate (smallest index on ties)
      for (int e0 = (tid >> 5) * 32; e0 < B * kUR; e0 += kCT) {  // warp-uniform: 16-lane groups = rows
        const int e = e0 + (tid & 31), b = e >> 4, r = e & 15, row = u * kUR + r;
        float v = -INFINITY;
        int vi = 0x7fffffff;
        if (b < B && row < R.V) {
          v = out[b * kUR + r];
          vi = R.voff + row;
          R.logits[(size_t)b * R.V + row] = v;
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
          const int i2 = __shfl_xor_sync(0xffffffffu, vi, o);
          if (v2 > v || (v2 == v && i2 < vi)) {
            v = v2;
            vi = i2;
          }
        }
        if (r == 0 && b < B) {  // one thread per row updates the row's running best
          if (u == u0 || v > S.lmv[b] || (v == S.lmv[b] && vi < S.lmi[b])) {
            S.lmv[b] = v;
            S.lmi[b] = vi;
          }
        }
      }
    }
  }
  if (u1 <= u0) return;
  if (tr) trace_ev(R, c, l, 29);
  cbar();
  if (kind == kLM && tid < B) R.cand[(size_t)c * kMaxB + tid] = ArgmaxCand{S.lmv[tid], S.lmi[tid]};
  cbar();
  if (tid == 0) {
    fence_ar();
    const unsigned long long old = atomicAdd(done, 1ull);
    *S.flag = kind == kLM && old + 1 == e1 * (unsigned long long)min(g.C, p.U);
    if (*S.flag) fence_ar();  // acquire: every CTA's candidate is visible to the argmax
  }
  cbar();
  if (kind == kLM) final_lm = *S.flag != 0;
}

// --------------------------------------------------------- row-parallel ---
// O / down: stream-K pieces; each pushes its [B][16] partial into every TP peer's LL slot
// (rank * 2 + piece) with tag epoch * n_phases + phase.
template <int NT, int FB>
__device__ void row_phase(const RankDev& R, const Geo& g, const Smem& S, int c, int l, int kind, uint32_t& it,
                          const __nv_bfloat16* src, int ld, uint32_t epv) {
  const Phase p = phase_of(R, g, kind, R.nq);
  const int Ce = row_ctas(p, g);
  if (c >= Ce) return;
  const int tid = threadIdx.x, B = g.B;
  const long long T = (long long)p.U * p.ns;
  const long long lo = rng_lo(c, T, Ce), hi = rng_lo(c + 1, T, Ce);
  const int phase = 2 * l + (kind == kDown ? 1 : 0);
  const uint64_t tag = (uint64_t)(epv * (uint32_t)g.n_phases + (uint32_t)phase) << 32;
  const long long pbase = (long long)(phase & 1) * R.ll_par_stride;
  Window W{1 << 30, -1, 0};
  Acc<NT, FB> acc;
#pragma unroll
  for (int q = 0; q < kAcc; ++q)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc.m[q][nt][0] = acc.m[q][nt][1] = acc.m[q][nt][2] = acc.m[q][nt][3] = 0.f;
#pragma unroll
  for (int b = 0; b < (FB > 0 ? FB : 1); ++b) acc.f[b] = 0.f;
  long long x = lo;
  while (x < hi) {
    const int u = (int)(x / p.ns), st0 = (int)(x % p.ns);
    const int st1 = (int)min((long long)p.ns, st0 + (hi - x));
    const int piece = st0 == 0 ? 0 : 1;
    mma_stages<NT, FB>(S, W, p, st0, st1, it, acc, 1, nullptr, nullptr, src, ld, B);
    reduce_unit<NT, FB>(S, acc, B);
    for (int e = tid; e < B * kUR; e += kCT) {
      const int b = e >> 4, r = e & 15;
      const uint64_t word = tag | (uint64_t)__float_as_uint(S.out[e]);
      const long long off = pbase + (long long)b * g.H + u * kUR + r;
      for (int q = 0; q < R.tp; ++q) {
        const int slot = (R.loopback ? q : R.rank) * 2 + piece;
        st_relaxed_sys_u64(R.ll_peer[q] + off + (long long)slot * R.ll_src_stride, word);
      }
    }
    x += st1 - st0;
  }
}

// ---------------------------------------------------------- norm slices ---
// Slice s (128 hidden columns) of norm instance j: resid += the TP ranks' pieces from the
// LL slots (j >= 1; phase j - 1), summed in (rank, piece) order, or resid = embedding (j == 0);
// publish the slice's sums of squares; one arrival on prog_norm[j] per slice. Every load of
// a slice is issued before any is waited on.
__device__ void norm_slices(const RankDev& R, const Geo& g, const Smem& S, int c, int j, uint32_t epv) {
  const int tid = threadIdx.x, B = g.B;
  const int s0 = span_lo(c, g.NS, g.C), s1 = span_lo(c + 1, g.NS, g.C);
  if (s0 >= s1) return;
  float* sq = R.sq[j & 1];
  float* sv = reinterpret_cast<float*>(S.scratch);  // [tp][16][128] per-rank sums
  const int tp = R.tp;
  const int phase = j - 1;
  const bool down = (phase & 1) != 0;
  const uint32_t want = epv * (uint32_t)g.n_phases + (uint32_t)phase;
  const int U = g.H / kUR, Ce = min(g.C, U);
  if (j > 0) cbar();  // the previous users of the scratch buffer are done
  for (int s = s0; s < s1; ++s) {
    const int k0 = s * 128;
    if (j > 0) {
      const int nit = tp * B * 64;  // (rank, row, column pair)
      for (int i0 = tid; i0 < nit; i0 += 2 * kCT) {
        ulonglong2 v[2][2];
        const uint64_t* pp[2];
        bool two[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int i = i0 + a * kCT;
          pp[a] = nullptr;
          two[a] = false;
          if (i < nit) {
            const int q = i / (B * 64), rem = i - q * (B * 64), b = rem >> 6, cp = rem & 63;
            const int u = (k0 + 2 * cp) / kUR;
            const int ns = ((down ? R.F : R.nq_of[q] * 128) + kSKu - 1) / kSKu;
            two[a] = unit_split(u, ns, U, Ce);
            pp[a] = R.ll_mine + (long long)(phase & 1) * R.ll_par_stride + (long long)(2 * q) * R.ll_src_stride +
                    (long long)b * g.H + k0 + 2 * cp;
            v[a][0] = ld_relaxed_sys_v2u64(pp[a]);
            if (two[a]) v[a][1] = ld_relaxed_sys_v2u64(pp[a] + R.ll_src_stride);
          }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int i = i0 + a * kCT;
          if (i >= nit) continue;
          float2 sum = make_float2(0.f, 0.f);
          for (int pc = 0; pc < (two[a] ? 2 : 1); ++pc) {
            ulonglong2 t = v[a][pc];
            if ((uint32_t)(t.x >> 32) != want || (uint32_t)(t.y >> 32) != want) {
              const uint64_t* p = pp[a] + pc * R.ll_src_stride;
              const uint64_t t0 = globaltimer_ns();
              do {
                bool fired = false;
                if (wait_abandoned(t0, &fired)) {
                  if (fired) {
                    printf("tps persist watchdog: LL phase %d block %d item %d piece %d tag %u != %u\n", phase,
                           blockIdx.x, i, pc, (unsigned)(t.x >> 32), want);
                    raise_abort(5);
                  }
                  break;
                }
                t = ld_relaxed_sys_v2u64(p);
              } while ((uint32_t)(t.x >> 32) != want || (uint32_t)(t.y >> 32) != want);
            }
            sum.x += __uint_as_float((uint32_t)t.x);
            sum.y += __uint_as_float((uint32_t)t.y);
          }
          const int q = i / (B * 64), rem = i - q * (B * 64), b = rem >> 6, cp = rem & 63;
          *reinterpret_cast<float2*>(sv + (q * kMaxB + b) * 128 + 2 * cp) = sum;
        }
      }
      cbar();
    }
    // residual update: thread (row b, column pair cp); rows in passes of kCW / 2 (2 warps a row)
    constexpr int kRowsPass = kCW / 2;
    for (int b0 = 0; b0 < B; b0 += kRowsPass) {
      const int b = b0 + (tid >> 6), cp = tid & 63;
      float ss = 0.f;
      if ((tid >> 6) < kRowsPass && b < B) {
        float* rp = R.resid + (size_t)b * g.H + k0 + 2 * cp;
        float2 x;
        if (j == 0) {
          x = __bfloat1622float2(
              *reinterpret_cast<const __nv_bfloat162*>(R.embed + (size_t)S.rtok[b] * g.H + k0 + 2 * cp));
        } else {
          float2 acc = make_float2(0.f, 0.f);
          for (int q = 0; q < tp; ++q) {
            const float2 t = *reinterpret_cast<const float2*>(sv + (q * kMaxB + b) * 128 + 2 * cp);
            acc.x += t.x;
            acc.y += t.y;
          }
          x = __ldcg(reinterpret_cast<const float2*>(rp));
          x.x += acc.x;
          x.y += acc.y;
        }
        *reinterpret_cast<float2*>(rp) = x;
        ss = x.x * x.x + x.y * x.y;
      }
      ss = warp_sum(ss);
      if ((tid & 31) == 0) S.wred[tid >> 5] = ss;
      cbar();
      if (tid < kRowsPass && b0 + tid < B) sq[s * kMaxB + b0 + tid] = S.wred[2 * tid] + S.wred[2 * tid + 1];
      cbar();
    }
    if (tid == 0) {
      fence_ar();
      atomicAdd(R.prog + 3 + j, 1ull);
    }
  }
}

__device__ void compute_rstd(const RankDev& R, const Geo& g, const Smem& S, int j) {
  const int tid = threadIdx.x;
  const float* sq = R.sq[j & 1];
  float* st = S.red;  // [NS][16] staged slice sums (one load per thread)
  for (int e = tid; e < g.NS * kMaxB; e += kCT) st[e] = (e & (kMaxB - 1)) < g.B ? __ldcg(sq + e) : 0.f;
  cbar();
  if (tid < kMaxB) {
    float s = 0.f;
    for (int i = 0; i < g.NS; ++i) s += st[i * kMaxB + tid];
    S.rstd[tid] = rsqrtf(s / (float)g.H + g.eps);
  }
  cbar();
}

// ------------------------------------------------------------ attention ---
// Units = (row b, KV head h, split s) with a per-row split count (>= kPagesPerSplit pages per
// split, at most the CTAs per (row, head)): S.rsa[b] splits, S.rub[b] the row's first unit.
constexpr int kPagesPerSplit = 2;

__device__ void attention(const RankDev& R, const Geo& g, const Smem& S, int c, int l) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = g.B, nkv = R.nkv;
  const int G = R.nq / nkv;
  const int nunits = S.rub[B];
  const int u0 = span_lo(c, nunits, g.C), u1 = span_lo(c + 1, nunits, g.C);
  __nv_bfloat16* stage = reinterpret_cast<__nv_bfloat16*>(S.scratch);  // 2 x (K [64][128] | V [64][128])
  int b = 0;
  for (int u = u0; u < u1; ++u) {
    while (u >= S.rub[b + 1]) ++b;
    const int Sa = S.rsa[b];
    const int h = (u - S.rub[b]) / Sa, s = (u - S.rub[b]) % Sa;
    const int slot = S.rslot[b];
    const int ctx = slot >= 0 ? S.rpos[b] + 1 : 0;
    const int npg = (ctx + kPage - 1) / kPage;
    const int p0 = (int)((long long)s * npg / Sa), p1 = (int)((long long)(s + 1) * npg / Sa);
    const __nv_bfloat16* kbase = R.kc[l];
    const __nv_bfloat16* vbase = R.vc[l];
    auto issue = [&](int p, int st) {
      const int page = R.page_table[(size_t)slot * R.max_pages + p];
      const __nv_bfloat16* kg = kbase + ((size_t)page * nkv + h) * kPage * 128;
      const __nv_bfloat16* vg = vbase + ((size_t)page * nkv + h) * kPage * 128;
      __nv_bfloat16* ks = stage + st * (2 * kPage * 128);
      __nv_bfloat16* vs = ks + kPage * 128;
      for (int ch = tid; ch < 1024; ch += kCT) {  // 1024 chunks of 16 B per tile
        const int t = ch >> 4, cc = ch & 15;
        cp_async16(ks + tile_off<128, false>(t, cc), kg + t * 128 + cc * 8);
        cp_async16(vs + tile_off<128, false>(t, cc), vg + t * 128 + cc * 8);
      }
    };
    uint32_t qa[8][4];
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    cbar();  // scratch free (previous unit's merge buffers read)
    trace_ev(R, c, l, 16);
    if (p0 < p1) issue(p0, 0);
    cp_async_commit();
    if (warp < 4) load_q_frags<128>(qa, R.q + ((size_t)b * R.nq + h * G) * 128, G);
    trace_ev(R, c, l, 17);
    for (int p = p0; p < p1; ++p) {
      const int st = (p - p0) & 1;
      if (p + 1 < p1) issue(p + 1, st ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
      cbar();
      if (warp < 4) {
        const __nv_bfloat16* ks = stage + st * (2 * kPage * 128);
        attend_page<128, false>(ks, ks + kPage * 128, qa, p * kPage, ctx, g.scale_log2, m_r, l_r, o);
      }
      cbar();
    }
    cp_async_wait<0>();
    trace_ev(R, c, l, 18);
    // merge the 4 warps' states -> unit partial (unnormalised O, running max M, sum L)
    float* wm = reinterpret_cast<float*>(S.scratch);  // [4][16]
    float* wl = wm + 64;                              // [4][16]
    float* wo = wl + 64;                              // [4][16][128]
    if (warp < 4) {
      const int gq = lane >> 2, cq = lane & 3;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
        l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
      }
      if (cq == 0) {
        wm[warp * 16 + gq] = m_r[0];
        wm[warp * 16 + gq + 8] = m_r[1];
        wl[warp * 16 + gq] = l_r[0];
        wl[warp * 16 + gq + 8] = l_r[1];
      }
#pragma unroll
      for (int dn = 0; dn < 16; ++dn) {
        const int d = dn * 8 + 2 * cq;
        *reinterpret_cast<float2*>(wo + (warp * 16 + gq) * 128 + d) = make_float2(o[dn][0], o[dn][1]);
        *reinterpret_cast<float2*>(wo + (warp * 16 + gq + 8) * 128 + d) = make_float2(o[dn][2], o[dn][3]);
      }
    }
    cbar();
    float* uo = R.att_o + (size_t)u * 16 * 128;
    for (int e = tid; e < G * 128; e += kCT) {
      const int r = e >> 7;
      float M = -INFINITY;
      for (int w2 = 0; w2 < 4; ++w2) M = fmaxf(M, wm[w2 * 16 + r]);
      float acc = 0.f, L = 0.f;
      if (M != -INFINITY)
        for (int w2 = 0; w2 < 4; ++w2) {
          const float f = exp2f(wm[w2 * 16 + r] - M);
          acc += wo[w2 * 2048 + e] * f;
          L += wl[w2 * 16 + r] * f;
        }
      uo[e] = acc;
      if ((e & 127) == 0) {
        R.att_m[(size_t)u * 16 + r] = M;
        R.att_l[(size_t)u * 16 + r] = L;
      }
    }
    cbar();
    trace_ev(R, c, l, 19);
    if (tid == 0) {
      fence_ar();
      unsigned int* cp = R.att_cnt + b * nkv + h;
      const unsigned int old = atomicAdd(cp, 1u);
      const bool last = old + 1 == (unsigned)Sa;
      if (last) {
        *cp = 0u;
        fence_ar();  // acquire: the other splits' partials
      }
      *S.flag = last ? 1 : 0;
    }
    cbar();
    trace_ev(R, c, l, 20);
    if (*S.flag) {
      const int ub = S.rub[b] + h * Sa;
      float* fm = reinterpret_cast<float*>(S.scratch);  // [16][kMaxSplit] split maxima -> weights
      float* fl = fm + 16 * kMaxSplit;                  // [16][kMaxSplit] split sums
      float* inv = fl + 16 * kMaxSplit;                 // [16] 1 / L
      for (int e = tid; e < G * Sa; e += kCT) {         // one batch: (row, split) per thread
        const int r = e / Sa, s2 = e - r * Sa;
        fm[r * kMaxSplit + s2] = __ldcg(R.att_m + (size_t)(ub + s2) * 16 + r);
        fl[r * kMaxSplit + s2] = __ldcg(R.att_l + (size_t)(ub + s2) * 16 + r);
      }
      cbar();
      trace_ev(R, c, l, 22);
      if (R.trace != nullptr && l == R.trace_layer && tid == 0) {
        R.trace[c * 32 + 25] = G * 100 + Sa;
      }
      if (tid < G) {
        float M = -INFINITY, L = 0.f;
        for (int s2 = 0; s2 < Sa; ++s2) M = fmaxf(M, fm[tid * kMaxSplit + s2]);
        for (int s2 = 0; s2 < Sa; ++s2) {
          const float f = M == -INFINITY ? 0.f : exp2f(fm[tid * kMaxSplit + s2] - M);
          fm[tid * kMaxSplit + s2] = f;
          L += fl[tid * kMaxSplit + s2] * f;
        }
        inv[tid] = L > 0.f ? 1.f / L : 0.f;
      }
      cbar();
      trace_ev(R, c, l, 23);
      // stage the splits' [G][128] partials in smem with cp.async (all loads in flight at once),
      // then thread (row, column) sums its splits in ascending order
      float* stg = fm + 8 * 1024 / 4;  // after the weight tables
      const int per = G * 128;         // floats per split
      const int cap = (kWinBytes - 8 * 1024) / (per * 4);
      float acc[(16 * 128 + kCT - 1) / kCT];
#pragma unroll
      for (int k = 0; k < (16 * 128 + kCT - 1) / kCT; ++k) acc[k] = 0.f;
      for (int sc0 = 0; sc0 < Sa; sc0 += cap) {
        const int nsc = min(cap, Sa - sc0);
        const int nch = nsc * per / 4;  // 16-byte chunks
        for (int ch = tid; ch < nch; ch += kCT) {
          const int s2 = ch / (per / 4), off = (ch - s2 * (per / 4)) * 4;
          cp_async16(stg + s2 * per + off, R.att_o + (size_t)(ub + sc0 + s2) * 16 * 128 + off);
        }
        cp_async_commit();
        cp_async_wait<0>();
        cbar();
#pragma unroll
        for (int k = 0; k < (16 * 128 + kCT - 1) / kCT; ++k) {
          const int e = tid + k * kCT;
          if (e < per) {
            const int r = e >> 7;
            float a2 = acc[k];
            for (int s2 = 0; s2 < nsc; ++s2) a2 += stg[s2 * per + e] * fm[r * kMaxSplit + sc0 + s2];
            acc[k] = a2;
          }
        }
        cbar();
      }
#pragma unroll
      for (int k = 0; k < (16 * 128 + kCT - 1) / kCT; ++k) {
        const int e = tid + k * kCT;
        if (e < per) {
          const int r = e >> 7, d = e & 127;
          R.attn[(size_t)b * R.nq * 128 + (h * G + r) * 128 + d] = f2bf(acc[k] * inv[r]);
        }
      }
      cbar();
      trace_ev(R, c, l, 21);
      if (tid == 0) {
        fence_ar();
        atomicAdd(R.prog + 3 + (2 * g.L + 1) + g.L + l, 1ull);
      }
    }
  }
}

// ------------------------------------------------------- final argmax ---
// Over the per-CTA candidates of the LM head (then, TP > 1, the ranks' candidates exchanged
// as LL pairs), smallest index on ties; writes the token, advances the row's position.
__device__ void finish_argmax(const RankDev& R, const Geo& g, const Smem& S, uint32_t epv) {
  const int tid = threadIdx.x, B = g.B;
  const int b = tid >> 3, part = tid & 7;  // 8 threads per row (128 of the consumer threads)
  const int nc = min(g.C, (R.V + kUR - 1) / kUR);
  float best = -INFINITY;
  int bidx = 0x7fffffff;
  if (b < B)
    for (int c0 = part; c0 < nc; c0 += 8 * 8) {
      ArgmaxCand t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int cc = c0 + u * 8;
        t[u] = ArgmaxCand{-INFINITY, 0x7fffffff};
        if (cc < nc) {
          const long long raw = __ldcg(reinterpret_cast<const long long*>(R.cand + (size_t)cc * kMaxB + b));
          t[u].val = __int_as_float((int)(raw & 0xffffffffll));
          t[u].idx = (int)(raw >> 32);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t[u].val > best || (t[u].val == best && t[u].idx < bidx)) {
          best = t[u].val;
          bidx = t[u].idx;
        }
    }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (v2 > best || (v2 == best && i2 < bidx)) {
      best = v2;
      bidx = i2;
    }
  }
  if (b >= B || part != 0) return;
  if (R.tp > 1) {
    const uint32_t want = epv * (uint32_t)g.n_phases + (uint32_t)(2 * g.L);
    const uint64_t tag = (uint64_t)want << 32;
    const int par = epv & 1;
    for (int q = 0; q < R.tp; ++q) {
      const int src = R.loopback ? q : R.rank;
      uint64_t* d = R.am_peer[q] + (((size_t)par * kMaxTP + src) * kMaxB + b) * 2;
      st_relaxed_sys_u64(d, tag | (uint64_t)__float_as_uint(best));
      st_relaxed_sys_u64(d + 1, tag | (uint64_t)(uint32_t)bidx);
    }
    ulonglong2 v[kMaxTP];
    for (int q = 0; q < R.tp; ++q) v[q] = ld_relaxed_sys_v2u64(R.am_mine + (((size_t)par * kMaxTP + q) * kMaxB + b) * 2);
    best = -INFINITY;
    bidx = 0x7fffffff;
    for (int q = 0; q < R.tp; ++q) {
      const uint64_t* p = R.am_mine + (((size_t)par * kMaxTP + q) * kMaxB + b) * 2;
      const uint64_t t0 = globaltimer_ns();
      while ((uint32_t)(v[q].x >> 32) != want || (uint32_t)(v[q].y >> 32) != want) {
        bool fired = false;
        if (wait_abandoned(t0, &fired)) {
          if (fired) {
            printf("tps persist watchdog: argmax src %d row %d\n", q, b);
            raise_abort(6);
          }
          break;
        }
        v[q] = ld_relaxed_sys_v2u64(p);
      }
      const float v2 = __uint_as_float((uint32_t)v[q].x);
      const int i2 = (int)(uint32_t)v[q].y;
      if (v2 > best || (v2 == best && i2 < bidx)) {
        best = v2;
        bidx = i2;
      }
    }
  }
  if (R.out_tok) R.out_tok[b] = bidx;
  const int slot = S.rslot[b];
  if (slot >= 0) {
    const int p = S.rpos[b];
    if ((R.prompt_len == nullptr || p + 1 >= R.prompt_len[slot]) && p + 1 < R.hist_ld)
      R.hist[(size_t)slot * R.hist_ld + p + 1] = bidx;
    R.pos[slot] = p + 1;
  }
}

// ------------------------------------------------------------------ kernel ---
template <int NT, int FB>
__global__ void __launch_bounds__(kThreads, 1) persist_step_kernel(const Ctx* __restrict__ ctx) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Geo g = ctx->g;
  const int rank_i = blockIdx.x / g.C, c = blockIdx.x % g.C;
  const RankDev& R = ctx->r[rank_i];
  // 1024-byte aligned by pointer arithmetic on the shared array (an integer round trip would
  // turn every smem access into a generic one)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Smem S;
  S.ring = base;
  S.scratch = base + kStages * kSlotBytes;
  S.red = reinterpret_cast<float*>(S.scratch + kWinBytes);
  S.out = reinterpret_cast<float*>(S.scratch + kWinBytes + kRedBytes);
  uint8_t* misc = S.scratch + kScratch;
  S.full = reinterpret_cast<uint64_t*>(misc);
  S.empty = S.full + kStages;
  S.rstd = reinterpret_cast<float*>(S.empty + kStages);
  S.flag = reinterpret_cast<int*>(S.rstd + kMaxB);
  S.rslot = S.flag + 4;
  S.rpos = S.rslot + kMaxB;
  S.rpage = S.rpos + kMaxB;
  S.rtok = S.rpage + kMaxB;
  S.rsa = S.rtok + kMaxB;
  S.rub = S.rsa + kMaxB;
  S.wred = reinterpret_cast<float*>(S.rub + kMaxB + 4);
  S.lmv = S.wred + kMaxB;
  S.lmi = reinterpret_cast<int*>(S.lmv + kMaxB);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], kCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == kCW) {
    if ((tid & 31) == 0) producer(R, g, c, S.ring, S.full, S.empty);
    return;
  }
  // every thread reads the step counters before any CTA can finish the step
  const unsigned long long e1 = *(volatile const unsigned long long*)R.prog + 1ull;
  // LL tags: the group epoch (TP > 1), else the step count + 1 (live tags never equal the
  // zero-initialised slots: tag = epoch * n_phases + phase >= n_phases)
  const uint32_t epv = (uint32_t)(R.ep ? *(volatile const uint64_t*)R.ep : e1);
  // per-row state of the step (row -> slot -> position -> page / token), read once
  if (tid < kMaxB) {
    const int slot = tid < g.B ? R.row_slot[tid] : -1;
    const int pos = slot >= 0 ? R.pos[slot] : 0;
    S.rslot[tid] = slot;
    S.rpos[tid] = pos;
    S.rpage[tid] = slot >= 0 ? R.page_table[(size_t)slot * R.max_pages + pos / kPage] : 0;
    S.rtok[tid] = slot >= 0 ? R.hist[(size_t)slot * R.hist_ld + pos] : 0;
    // attention splits: >= kPagesPerSplit pages each, at most the CTAs per (row, KV head)
    const int smax = max(1, min(kMaxSplit, g.C / max(1, g.B * R.nkv)));
    const int npg = slot >= 0 ? (pos + 1 + kPage - 1) / kPage : 0;
    S.rsa[tid] = max(1, min(smax, (npg + kPagesPerSplit - 1) / kPagesPerSplit));
  }
  cbar();
  if (tid == 0) {
    int acc = 0;
    for (int b = 0; b < g.B; ++b) {
      S.rub[b] = acc;
      acc += S.rsa[b] * R.nkv;
    }
    S.rub[g.B] = acc;
  }
  cbar();
  unsigned long long* prog_norm = R.prog + 3;
  unsigned long long* prog_qkv = prog_norm + 2 * g.L + 1;
  unsigned long long* prog_att = prog_qkv + g.L;
  unsigned long long* prog_act = prog_att + g.L;
  const int act_qkv = min(g.C, phase_of(R, g, kQKV, R.nq).U);  // CTAs with units (one arrival each)
  const int act_gu = min(g.C, phase_of(R, g, kGU, R.nq).U);
  uint32_t it = 0;
  bool final_lm = false;
  trace_ev(R, c, 0, 13);
  norm_slices(R, g, S, c, 0, epv);
  for (int l = 0; l < g.L; ++l) {
    trace_ev(R, c, l, 0);
    cwait(prog_norm + 2 * l, e1 * (unsigned long long)g.NS, 1);
    trace_ev(R, c, l, 1);
    compute_rstd(R, g, S, 2 * l);
    col_phase<NT, FB>(R, g, S, c, l, kQKV, it, R.resid, R.ln1[l], prog_qkv + l, e1, final_lm);
    trace_ev(R, c, l, 2);
    cwait(prog_qkv + l, e1 * (unsigned long long)act_qkv, 2);
    trace_ev(R, c, l, 3);
    attention(R, g, S, c, l);
    trace_ev(R, c, l, 4);
    // attention merges count B * nkv per step; the step's end pads the counter to kMaxB * nkv
    // so targets stay a function of the step when the bucket changes between steps
    cwait(prog_att + l, (e1 - 1ull) * (unsigned long long)(kMaxB * R.nkv) + (unsigned long long)(g.B * R.nkv), 3);
    trace_ev(R, c, l, 5);
    row_phase<NT, FB>(R, g, S, c, l, kO, it, R.attn, R.nq * 128, epv);
    trace_ev(R, c, l, 6);
    norm_slices(R, g, S, c, 2 * l + 1, epv);
    trace_ev(R, c, l, 7);
    cwait(prog_norm + 2 * l + 1, e1 * (unsigned long long)g.NS, 4);
    trace_ev(R, c, l, 8);
    compute_rstd(R, g, S, 2 * l + 1);
    col_phase<NT, FB>(R, g, S, c, l, kGU, it, R.resid, R.ln2[l], prog_act + l, e1, final_lm);
    trace_ev(R, c, l, 9);
    cwait(prog_act + l, e1 * (unsigned long long)act_gu, 5);
    trace_ev(R, c, l, 10);
    row_phase<NT, FB>(R, g, S, c, l, kDown, it, R.act, R.F, epv);
    trace_ev(R, c, l, 11);
    norm_slices(R, g, S, c, 2 * l + 2, epv);
    trace_ev(R, c, l, 12);
  }
  cwait(prog_norm + 2 * g.L, e1 * (unsigned long long)g.NS, 6);
  compute_rstd(R, g, S, 2 * g.L);
  col_phase<NT, FB>(R, g, S, c, g.L, kLM, it, R.resid, R.ln_f, R.prog + 2, e1, final_lm);
  if (final_lm) finish_argmax(R, g, S, epv);
  trace_ev(R, c, 0, 14);
  cbar();
  if (tid == 0) {
    fence_ar();
    const unsigned long long old = atomicAdd(R.prog + 1, 1ull);
    if (old + 1 == (unsigned long long)g.C) {  // the rank's last CTA: advance the step
      R.prog[1] = 0ull;
      if (R.ctr)
        for (int ph = 0; ph < g.n_phases; ++ph) atomicAdd(R.ctr + ph, (unsigned long long)R.tp);
      if (R.ep_adv) *R.ep_adv += 1ull;
      for (int l = 0; l < g.L; ++l) prog_att[l] += (unsigned long long)((kMaxB - g.B) * R.nkv);
      fence_ar();
      atomicAdd(R.prog, 1ull);
    }
  }
}

// ------------------------------------------------------------------- host ---
struct WorkLayout {
  size_t prog, att_cnt, resid, q, attn, act, att_o, att_m, att_l, sq0, sq1, cand, ll, total;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static int max_units(int C, int nkv) { return std::max(C, kMaxB * nkv) + kMaxSplit; }

static WorkLayout work_layout(const tps_persist_geom& g, const tps_persist_rank& r, int C) {
  WorkLayout w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const int L = g.num_layers, H = g.hidden;
  const int mu = max_units(C, r.nkv);
  w.prog = take(8 * (3 + (2 * L + 1) + 3 * L));
  w.att_cnt = take(4 * (size_t)kMaxB * r.nkv);
  w.resid = take(4 * (size_t)kMaxB * H);
  w.q = take(2 * (size_t)kMaxB * r.nq * 128);
  w.attn = take(2 * (size_t)kMaxB * r.nq * 128);
  w.act = take(2 * (size_t)kMaxB * r.ffn);
  w.att_o = take(4 * (size_t)mu * 16 * 128);
  w.att_m = take(4 * (size_t)mu * 16);
  w.att_l = take(4 * (size_t)mu * 16);
  w.sq0 = take(4 * (size_t)(H / 128) * kMaxB);
  w.sq1 = take(4 * (size_t)(H / 128) * kMaxB);
  w.cand = take(8 * (size_t)C * kMaxB);
  w.ll = take(8 * (size_t)2 * 2 * kMaxB * H);  // local LL area (tp == 1): [2 parity][2 pieces][16 rows][H]
  w.total = off;
  return w;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Row-major bf16 [rows][cols] viewed as 3-D {64, rows, cols / 64} with strides {2 * cols, 128}:
// a box {64, box_rows, 32 KB / (box_rows * 128)} lands in smem as [chunk][row][64], each 128-byte
// row swizzled by its row index (SWIZZLE_128B), so ldmatrix over 8 rows is conflict-free.
static int make_tmap3(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  if (!fn) return fail(kCuda, "cuTensorMapEncodeTiled entry point unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || cols % 64 != 0)
    return fail(kInvalid, "persist tensor map: 16-byte aligned base and a multiple of 64 columns");
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)(kSlotBytes / (box_rows * 128))};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(kCuda, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
  return kOk;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

static bool smem_configured = false;
static std::mutex cfg_mu;

static int configure() {
  std::lock_guard<std::mutex> lk(cfg_mu);
  if (smem_configured) return kOk;
  TPS_CUDA_TRY(cudaFuncSetAttribute(persist_step_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  TPS_CUDA_TRY(cudaFuncSetAttribute(persist_step_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  TPS_CUDA_TRY(cudaFuncSetAttribute(persist_step_kernel<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  TPS_CUDA_TRY(cudaFuncSetAttribute(persist_step_kernel<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  TPS_CUDA_TRY(cudaFuncSetAttribute(persist_step_kernel<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
  smem_configured = true;
  return kOk;
}

}  // namespace pst

int configure_persist() { return pst::configure(); }

}  // namespace tps

using namespace tps;
using namespace tps::pst;

extern "C" {

int64_t tps_persist_struct_bytes(int which) {
  return which == 0 ? (int64_t)sizeof(tps_persist_geom) : which == 1 ? (int64_t)sizeof(tps_persist_rank) : -1;
}

int tps_persist_supported(const tps_persist_geom* g, const tps_persist_rank* r, int B) {
  if (!g || !r) return 0;
  if (g->head_dim != 128 || B < 1 || B > kMaxB) return 0;
  if (g->hidden % 128 || g->hidden > 16384) return 0;
  if (r->ffn % 64 || r->nkv < 1 || r->nq % r->nkv || r->nq / r->nkv > 16 || r->vocab < kUR) return 0;
  if (r->tp < 1 || r->tp > kMaxTP) return 0;
  return 1;
}

int64_t tps_persist_work_bytes(const tps_persist_geom* g, const tps_persist_rank* r, int ctas) {
  if (!g || !r || ctas < 1) return -1;
  return (int64_t)work_layout(*g, *r, ctas).total;
}

int64_t tps_persist_ctx_bytes(const tps_persist_geom* g, int nranks) {
  if (!g || nranks < 1) return -1;
  const size_t head = align_up(offsetof(Ctx, r) + sizeof(RankDev) * nranks, 128);
  const size_t per = align_up((size_t)(4 * g->num_layers + 1) * sizeof(CUtensorMap), 128) +
                     align_up((size_t)5 * g->num_layers * sizeof(void*), 128);
  return (int64_t)(head + per * nranks);
}

int tps_persist_prepare(const tps_persist_geom* gp, const tps_persist_rank* ranks, int nranks, int B, int ctas,
                        void* dev_ctx, void* stream) {
  TPS_CHECK_ARG(gp && ranks && nranks >= 1 && nranks <= kMaxTP && dev_ctx && ctas >= 1, "persist_prepare: arguments");
  const tps_persist_geom& g = *gp;
  for (int i = 0; i < nranks; ++i)
    TPS_CHECK_ARG(tps_persist_supported(gp, ranks + i, B), "persist_prepare: unsupported shape");
  TPS_CHECK_ARG(ctas * nranks <= kNumSMs, "persist_prepare: more CTAs than SMs");
  int rc = configure();
  if (rc) return rc;
  const int L = g.num_layers;
  const size_t bytes = (size_t)tps_persist_ctx_bytes(gp, nranks);
  std::vector<uint8_t> host(bytes, 0);
  const size_t head = align_up(offsetof(Ctx, r) + sizeof(RankDev) * nranks, 128);
  const size_t tm_bytes = align_up((size_t)(4 * L + 1) * sizeof(CUtensorMap), 128);
  const size_t per = tm_bytes + align_up((size_t)5 * L * sizeof(void*), 128);
  Geo geo{};
  geo.L = L;
  geo.H = g.hidden;
  geo.B = B;
  geo.C = ctas;
  geo.nranks = nranks;
  geo.n_phases = g.n_phases;
  geo.NS = g.hidden / 128;
  geo.eps = g.rms_eps;
  geo.scale_log2 = 1.4426950408889634f / sqrtf(128.f);
  const int nkv = ranks[0].nkv;
  for (int i = 0; i < nranks; ++i)
    TPS_CHECK_ARG(ranks[i].nkv == nkv, "persist_prepare: ranks of a group differ in KV heads");
  geo.S_att = std::max(1, std::min(kMaxSplit, ctas / std::max(1, B * nkv)));
  geo.max_units = max_units(ctas, nkv);
  TPS_CHECK_ARG(B * nkv * geo.S_att <= geo.max_units, "persist_prepare: attention units");
  std::memcpy(host.data(), &geo, sizeof(Geo));
  uint8_t* dbase = reinterpret_cast<uint8_t*>(dev_ctx);
  for (int i = 0; i < nranks; ++i) {
    const tps_persist_rank& r = ranks[i];
    uint8_t* hblk = host.data() + head + per * i;
    uint8_t* dblk = dbase + head + per * i;
    CUtensorMap* tm = reinterpret_cast<CUtensorMap*>(hblk);
    const int64_t H = g.hidden;
    for (int l = 0; l < L; ++l) {
      const int64_t nqkv = (int64_t)(r.nq + 2 * r.nkv) * 128, kq = (int64_t)r.nq * 128;
      // paired units (QKV, gate/up) load 8-row boxes, the others 16-row boxes
      rc = make_tmap3(&tm[4 * l + 0], r.w_qkv[l], nqkv, H, 8);
      if (!rc) rc = make_tmap3(&tm[4 * l + 1], r.w_o[l], H, kq, kUR);
      if (!rc) rc = make_tmap3(&tm[4 * l + 2], r.w_gu[l], 2 * (int64_t)r.ffn, H, 8);
      if (!rc) rc = make_tmap3(&tm[4 * l + 3], r.w_d[l], H, r.ffn, kUR);
      if (rc) return rc;
    }
    rc = make_tmap3(&tm[4 * L], r.lm_head, r.vocab, H, kUR);
    if (rc) return rc;
    const void** ptrs = reinterpret_cast<const void**>(hblk + tm_bytes);
    for (int l = 0; l < L; ++l) {
      ptrs[0 * L + l] = r.b_qkv ? r.b_qkv[l] : nullptr;
      ptrs[1 * L + l] = r.ln1[l];
      ptrs[2 * L + l] = r.ln2[l];
      ptrs[3 * L + l] = r.k_cache[l];
      ptrs[4 * L + l] = r.v_cache[l];
    }
    void* const* dptrs = reinterpret_cast<void* const*>(dblk + tm_bytes);
    RankDev d{};
    d.tmaps = reinterpret_cast<const CUtensorMap*>(dblk);
    d.b_qkv = reinterpret_cast<const __nv_bfloat16* const*>(dptrs + 0 * L);
    d.ln1 = reinterpret_cast<const __nv_bfloat16* const*>(dptrs + 1 * L);
    d.ln2 = reinterpret_cast<const __nv_bfloat16* const*>(dptrs + 2 * L);
    d.kc = reinterpret_cast<__nv_bfloat16* const*>(dptrs + 3 * L);
    d.vc = reinterpret_cast<__nv_bfloat16* const*>(dptrs + 4 * L);
    d.embed = static_cast<const __nv_bfloat16*>(r.embed);
    d.ln_f = static_cast<const __nv_bfloat16*>(r.ln_f);
    d.nq = r.nq;
    d.nkv = r.nkv;
    d.F = r.ffn;
    d.V = r.vocab;
    d.voff = r.vocab_off;
    d.row_slot = r.row_slot;
    d.pos = r.pos;
    d.page_table = r.page_table;
    d.max_pages = r.max_pages;
    d.hist = r.history;
    d.hist_ld = r.hist_ld;
    d.prompt_len = r.prompt_len;
    d.out_tok = r.out_tok;
    d.cos_t = r.cos_t;
    d.sin_t = r.sin_t;
    TPS_CHECK_ARG(r.work && r.work_bytes >= (int64_t)work_layout(g, r, ctas).total, "persist_prepare: work buffer");
    const WorkLayout w = work_layout(g, r, ctas);
    uint8_t* wb = static_cast<uint8_t*>(r.work);
    d.prog = reinterpret_cast<unsigned long long*>(wb + w.prog);
    d.att_cnt = reinterpret_cast<unsigned int*>(wb + w.att_cnt);
    d.resid = reinterpret_cast<float*>(wb + w.resid);
    d.q = reinterpret_cast<__nv_bfloat16*>(wb + w.q);
    d.attn = reinterpret_cast<__nv_bfloat16*>(wb + w.attn);
    d.act = reinterpret_cast<__nv_bfloat16*>(wb + w.act);
    d.att_o = reinterpret_cast<float*>(wb + w.att_o);
    d.att_m = reinterpret_cast<float*>(wb + w.att_m);
    d.att_l = reinterpret_cast<float*>(wb + w.att_l);
    d.sq[0] = reinterpret_cast<float*>(wb + w.sq0);
    d.sq[1] = reinterpret_cast<float*>(wb + w.sq1);
    d.cand = reinterpret_cast<ArgmaxCand*>(wb + w.cand);
    TPS_CHECK_ARG(r.logits, "persist_prepare: logits buffer");
    d.logits = r.logits;
    d.tp = r.tp;
    d.rank = r.rank;
    d.loopback = r.loopback;
    TPS_CHECK_ARG(r.tp <= kMaxTP && 2 * r.tp <= 16, "persist_prepare: tp");
    for (int q = 0; q < kMaxTP; ++q)  // loopback: this rank's own shapes play every peer
      d.nq_of[q] = (q < r.tp && !r.loopback && r.nq_of[q] > 0) ? r.nq_of[q] : r.nq;
    if (r.tp == 1) {
      uint64_t* ll = reinterpret_cast<uint64_t*>(wb + w.ll);
      d.ll_par_stride = 2LL * kMaxB * g.hidden;
      d.ll_src_stride = (long long)kMaxB * g.hidden;
      d.ll_peer[0] = ll;
      d.ll_mine = ll;
      d.ep = nullptr;       // tags from the step counter
      d.ep_adv = nullptr;
      d.ctr = nullptr;
    } else {
      TPS_CHECK_ARG(r.ll_mine && r.am_mine && r.epoch, "persist_prepare: TP exchange buffers");
      d.ll_par_stride = r.ll_par_stride;
      d.ll_src_stride = r.ll_src_stride;
      for (int q = 0; q < r.tp; ++q) {
        TPS_CHECK_ARG(r.ll_peer[q] && r.am_peer[q], "persist_prepare: peer tables");
        d.ll_peer[q] = r.ll_peer[q];
        d.am_peer[q] = r.am_peer[q];
      }
      d.ll_mine = r.ll_mine;
      d.am_mine = r.am_mine;
      d.ep = r.epoch;
      d.ep_adv = r.epoch;
      d.ctr = reinterpret_cast<unsigned long long*>(r.ctr);
    }
    d.trace = reinterpret_cast<unsigned long long*>(r.trace);
    d.trace_layer = r.trace_layer;
    std::memcpy(host.data() + offsetof(Ctx, r) + sizeof(RankDev) * i, &d, sizeof(RankDev));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TPS_CUDA_TRY(cudaMemcpyAsync(dev_ctx, host.data(), bytes, cudaMemcpyHostToDevice, st));
  TPS_CUDA_TRY(cudaStreamSynchronize(st));
  return kOk;
}

int tps_persist_launch(const void* dev_ctx, int nranks, int ctas, int B, void* stream) {
  TPS_CHECK_ARG(dev_ctx && nranks >= 1 && ctas >= 1 && B >= 1 && B <= kMaxB, "persist_launch: arguments");
  int rc = configure();
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nranks * ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const Ctx* c = static_cast<const Ctx*>(dev_ctx);
  // B <= 4: CUDA-core GEMV (FB rows); else the m16n8k16 tensor form with 1 or 2 n-tiles
  const int fb = env_int("TPS_PERSIST_FMA_MAX", 4);
  cudaError_t e;
  if (B <= 1 && fb >= 1) e = cudaLaunchKernelEx(&cfg, persist_step_kernel<1, 1>, c);
  else if (B <= 2 && fb >= 2) e = cudaLaunchKernelEx(&cfg, persist_step_kernel<1, 2>, c);
  else if (B <= 4 && fb >= 4) e = cudaLaunchKernelEx(&cfg, persist_step_kernel<1, 4>, c);
  else if (B <= 8) e = cudaLaunchKernelEx(&cfg, persist_step_kernel<1, 0>, c);
  else e = cudaLaunchKernelEx(&cfg, persist_step_kernel<2, 0>, c);
  if (e != cudaSuccess) return fail(kCuda, std::string("persist launch: ") + cudaGetErrorString(e));
  return kOk;
}

}  // extern "C"
