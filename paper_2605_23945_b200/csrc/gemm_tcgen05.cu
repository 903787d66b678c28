// Skinny decode GEMM on 5th-gen tensor cores (tcgen05 + TMA + TMEM), sm_100a.
//
//   out[split][b][n] = sum_{k in split} W[n][k] * X[b][k]        (fp32 partials)
//
// This is the Infer Executor's column-/row-parallel projection (QKV, O, gate/up,
// down, LM head) for a decode step, i.e. the work the reference prices with the
// HBM/compute terms of oracle_decode_latency (tpshift/latency.py:123-124).
// Decode is weight-streaming bound (batch B <= 256 << the bf16 ridge), so the
// kernel is built to keep HBM busy:
//   * swap-AB: the weight tile is the 128-row UMMA "M" operand, the B tokens are
//     the UMMA "N" operand (N = BN, padded to a multiple of 16), so one MMA
//     shape serves every batch from 1 to 256;
//   * persistent grid (<= 148 CTAs, one per SM) walking (tile, k-split) units;
//     k-splits fill the machine when N/128 tiles alone would not;
//   * warp-specialised: warp0 = TMA producer (weights EVICT_FIRST, activations
//     EVICT_LAST), warp1 = single-thread tcgen05.mma issuer, warp2 = TMEM
//     allocator, warps4-7 = epilogue (tcgen05.ld -> fp32 partials);
//   * a 4-8 stage smem ring (SWIZZLE_128B) and two TMEM accumulators so the
//     epilogue of unit i overlaps the MMAs of unit i+1.
// Split partials are reduced, in fixed split order, by the consumer kernels
// (norm / rope / silu / argmax), which keeps results deterministic.
#include <cooperative_groups.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "decode_ops.cuh"

namespace tps {

constexpr int kBM = 128;  // weight rows per tile == UMMA M
constexpr int kBK = 64;   // K elements per stage == one 128-byte swizzle row
constexpr int kGemmThreads = 256;

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStagesRaw = (200 * 1024) / kStageBytes;
#ifndef TPS_GEMM_MAX_STAGES
#define TPS_GEMM_MAX_STAGES 8
#endif
  static constexpr int kStages = kStagesRaw > TPS_GEMM_MAX_STAGES ? TPS_GEMM_MAX_STAGES : kStagesRaw;
  static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int kBarBytes = 256;
  static constexpr int kEpiBytes = 64 * 17 * 4;  // SwiGLU epilogue exchange buffer
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kBarBytes + kEpiBytes;
  // the cluster-reduced form keeps a shallower ring so two CTAs fit per SM: the next
  // launch's clusters become resident (and prefetch) while this one drains
#ifndef TPS_CLUSTER_STAGES
#define TPS_CLUSTER_STAGES 4
#endif
  static constexpr int kClusterStages = kStages < TPS_CLUSTER_STAGES ? kStages : TPS_CLUSTER_STAGES;
  static constexpr int kClusterSmemBytes = 1024 + kClusterStages * kStageBytes + kBarBytes + kEpiBytes;
  static_assert(BN * kBM * 4 <= kClusterStages * kStageBytes, "the partial tile must fit the drained ring");
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128 must be 16..256, %16");
  static_assert(kStages >= 3, "need at least 3 stages");
};

// UMMA shared-memory descriptor, K-major operand in the canonical SWIZZLE_128B layout
// (8-row x 128-byte atoms; SBO = 1024 B between atoms; version 1 for sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue modes: kEpiPartial writes fp32 split-K partials [split][B][N]; kEpiSiluMul
// (splits == 1, gate/up weights stored as interleaved 64-row blocks [gate c | up c])
// writes act[b][f] = bf16(silu(gate) * up) directly -- the SwiGLU never round-trips HBM.
constexpr int kEpiPartial = 0;
constexpr int kEpiSiluMul = 1;
// kEpiClusterLL: row-parallel projection + TP allreduce push. The split-K CTAs of a tile
// (one cluster) sum their partials over DSMEM in split order and push ONE LL {value, tag}
// pair per element to every peer (tps_linear_push_ll pushes every split partial: S x the
// NVLink bytes and tp x S sources for the consumer; tps_reduce_push_ll needs a launch).
constexpr int kEpiClusterLL = 3;
// kEpiArgmax: LM head (splits == 1): the fp32 logits as kEpiPartial, plus the greedy candidate
// {max logit, smallest index on ties} of every (row, 128-column tile) -- argmax stage 1 done
// in the epilogue, so no kernel re-reads the logits (tps_argmax_finalize merges the tiles).
constexpr int kEpiArgmax = 6;

struct ArgEpi {
  ArgmaxCand* cand;  // [rows][ntiles]
  int ntiles;
  int vocab0;        // global index of column 0
};
constexpr bool cluster_epi(int epi) { return epi == kEpiClusterLL; }


namespace cg = cooperative_groups;

// Finishing of kEpiClusterLL (all 256 threads of every CTA of the cluster): CTA s of S sums
// columns [s*128/S, (s+1)*128/S) of the tile. part: this CTA's [BN][128] fp32 tile partial
// (row j = token row, column r = weight row).
template <int BN>
__device__ __forceinline__ void cluster_ll_finish(const float* part, const DstList& dst, uint64_t tag, int tile,
                                                  int N, int rows) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();  // every split's partial tile is parked in its CTA's smem
  const int S = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int r0 = rank * kBM / S, r1 = (rank + 1) * kBM / S;
  const int nr = r1 - r0;
  const float* rp[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) rp[s] = s < S ? cl.map_shared_rank(part, s) : part;
  for (int it = threadIdx.x; it < nr * rows; it += kGemmThreads) {
    const int r = r0 + it % nr, j = it / nr;
    const int n = tile * kBM + r;
    if (n >= N) continue;
    float v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s)
      if (s < S) v[s] = rp[s][j * kBM + r];
    float x = 0.f;  // split order, from 0 (as tps_reduce_push_ll)
#pragma unroll
    for (int s = 0; s < 16; ++s)
      if (s < S) x += v[s];
    if (tag)
      for (int d = 0; d < dst.n; ++d)
        st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(dst.p[d]) + (size_t)j * N + n, tag | __float_as_uint(x));
    else
      dst.p[0][(size_t)j * N + n] = x;  // local fp32 result (tag 0: not issued by the library)
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_swapab_kernel(const __grid_constant__ CUtensorMap tmap_w,
                       const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ DstList dst,
                       long long split_stride, int N, int B, int num_tiles, int splits, int chunks, int acts,
                       __nv_bfloat16* __restrict__ act_out, int ld_act, const __grid_constant__ SignalSpec sig,
                       const uint64_t* __restrict__ tag_epoch, uint32_t tag_mult, uint32_t tag_add,
                       const __grid_constant__ ArgEpi arg) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = cluster_epi(EPI) ? Cfg::kClusterStages : Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  float* up_buf = reinterpret_cast<float*>(smem + S * Cfg::kStageBytes + Cfg::kBarBytes);  // [64][17]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tmem_full = bars + 2 * S;
  uint64_t* tmem_empty = bars + 2 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

  const unsigned int trs =
      trace_begin(EPI == kEpiSiluMul ? kTrGemmSilu : EPI == kEpiClusterLL ? kTrGemmPush : kTrGemm);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // unit u = ((tile * splits + split) * acts + act): the activation tiles of one weight
  // chunk range run on neighbouring CTAs at the same time, so L2 dedups the weight stream
  const int units = num_tiles * splits * acts;
  auto unit_of = [&](int u, int& tile, int& act, int& c0, int& c1) {
    act = u % acts;
    const int ts = u / acts;
    tile = ts / splits;
    const int split = ts % splits;
    c0 = (int)((long long)split * chunks / splits);
    c1 = (int)((long long)(split + 1) * chunks / splits);
    return split;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_w);
    prefetch_tmap(&tmap_x);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  if (warp >= 4) pdl_wait();  // epilogue writes the partial buffer the predecessor may still read

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      // Weights are never produced by the preceding decode kernels: stream the
      // first unit's weight tiles into the ring *before* the programmatic
      // dependency wait, so this kernel's HBM stream starts while its
      // predecessor is still running; only the activation loads wait.
      int pre = 0;
      if ((int)blockIdx.x < units) {
        int tile, act, c0, c1;
        unit_of(blockIdx.x, tile, act, c0, c1);
        pre = min(S, c1 - c0);
        for (int i = 0; i < pre; ++i) {
          mbar_arrive_expect_tx(&full[i], Cfg::kStageBytes);
          tma_load_2d(smem_a + i * Cfg::kABytes, &tmap_w, &full[i], (c0 + i) * kBK, tile * kBM, pol_w);
        }
        pdl_wait();
        trace_mark(trs, 2);
        for (int i = 0; i < pre; ++i)
          tma_load_2d(smem_b + i * Cfg::kBBytes, &tmap_x, &full[i], (c0 + i) * kBK, act * BN, pol_x);
        stage = pre % S;
        phase = (pre == S) ? 1u : 0u;
      } else {
        pdl_wait();
      }
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int tile, act, c0, c1;
        unit_of(u, tile, act, c0, c1);
        for (int c = (u == (int)blockIdx.x ? c0 + pre : c0); c < c1; ++c) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
          tma_load_2d(smem_a + stage * Cfg::kABytes, &tmap_w, &full[stage], c * kBK, tile * kBM, pol_w);
          tma_load_2d(smem_b + stage * Cfg::kBBytes, &tmap_x, &full[stage], c * kBK, act * BN, pol_x);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread) ----------------
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(kBM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int tile, act, c0, c1;
        unit_of(u, tile, act, c0, c1);
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int c = c0; c < c1; ++c) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a0 = umma_desc_sw128(smem_u32(smem_a + stage * Cfg::kABytes));
          const uint64_t b0 = umma_desc_sw128(smem_u32(smem_b + stage * Cfg::kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // advance 16 bf16 = 32 bytes along K inside the 128-byte swizzle row
            umma_bf16(d_tmem, a0 + (uint64_t)(2 * k), b0 + (uint64_t)(2 * k), idesc,
                      (c > c0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tmem_full[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> fp32 partials ----------------
    const int q = warp & 3;  // TMEM lane quadrant owned by this warp
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int tile, act, c0, c1;
      const int split = unit_of(u, tile, act, c0, c1);
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int n = tile * kBM + q * 32 + lane;
      const int b0 = act * BN;
      const int rows = min(BN, B - b0);
      if constexpr (EPI == kEpiPartial || EPI == kEpiArgmax) {
        // fp32 partial of (split, rows b0.., column n) into every destination: the local
        // split-K workspace, or -- the fused TP allreduce -- this rank's slots in each
        // peer's receive area (NVLink P2P stores), split-major with split_stride. The
        // consumer sums the partials in a fixed order (deterministic, no atomics).
        // LL mode (tag_epoch set): every element goes out as one 8-byte {value, tag} store
        // (tag = epoch * mult + add), so the consumer polls the data itself -- no fence,
        // counter or last-CTA signal on the critical path (NCCL's LL protocol).
        const size_t off = (size_t)split * (size_t)split_stride + (size_t)b0 * (size_t)N + (size_t)n;
        const uint64_t tag = tag_epoch ? ((uint64_t)((uint32_t)(*(volatile const uint64_t*)tag_epoch * tag_mult +
                                                                tag_add)) << 32) : 0ull;
        for (int j0 = 0; j0 < rows; j0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem_base + (uint32_t)(acc * BN + j0) + ((uint32_t)(q * 32) << 16), r);
          if (n < N) {
            for (int d = 0; d < dst.n; ++d) {
              if (tag_epoch) {
                uint64_t* o = reinterpret_cast<uint64_t*>(dst.p[d]) + off;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (j0 + j < rows) st_relaxed_sys_u64(o + (size_t)(j0 + j) * N, tag | r[j]);
              } else {
                float* o = dst.p[d] + off;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (j0 + j < rows) o[(size_t)(j0 + j) * N] = __uint_as_float(r[j]);
              }
            }
          }
          if constexpr (EPI == kEpiArgmax) {
            // per row: warp max over its 32 columns (smallest index on ties), then the 4 warps
            ArgmaxCand* xb = reinterpret_cast<ArgmaxCand*>(up_buf);  // [4][16]
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float v = (n < N) ? __uint_as_float(r[j]) : -INFINITY;
              int ix = arg.vocab0 + n;
#pragma unroll
              for (int o2 = 16; o2 > 0; o2 >>= 1) {
                const float v2 = __shfl_xor_sync(0xffffffffu, v, o2);
                const int i2 = __shfl_xor_sync(0xffffffffu, ix, o2);
                if (v2 > v || (v2 == v && i2 < ix)) {
                  v = v2;
                  ix = i2;
                }
              }
              if (lane == 0) xb[q * 16 + j] = ArgmaxCand{v, ix};
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (q == 0 && lane < 16 && j0 + lane < rows) {
              ArgmaxCand best = xb[lane];
#pragma unroll
              for (int w = 1; w < 4; ++w) {
                const ArgmaxCand c = xb[w * 16 + lane];
                if (c.val > best.val || (c.val == best.val && c.idx < best.idx)) best = c;
              }
              arg.cand[(size_t)(b0 + j0 + lane) * arg.ntiles + tile] = best;
            }
            asm volatile("bar.sync 2, 128;" ::: "memory");
          }
        }
      } else if constexpr (cluster_epi(EPI)) {
        // one unit per CTA: its MMAs (and so every smem read of the ring) are complete
        float* part = reinterpret_cast<float*>(smem);
        const int r = q * 32 + lane;
        for (int j0 = 0; j0 < rows; j0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem_base + (uint32_t)(acc * BN + j0) + ((uint32_t)(q * 32) << 16), v);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j0 + j < rows) part[(j0 + j) * kBM + r] = __uint_as_float(v[j]);
        }
      } else {
        // rows 0..63 of the tile are gate(f), rows 64..127 up(f), f = tile*64 + row
        const int m = (q & 1) * 32 + lane;
        const int f = tile * 64 + m;
        const int F = N / 2;
        for (int j0 = 0; j0 < rows; j0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem_base + (uint32_t)(acc * BN + j0) + ((uint32_t)(q * 32) << 16), r);
          if (q >= 2) {
#pragma unroll
            for (int j = 0; j < 16; ++j) up_buf[m * 17 + j] = __uint_as_float(r[j]);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (q < 2 && f < F) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j0 + j < rows) {
                const float g = __uint_as_float(r[j]);
                const float u = up_buf[m * 17 + j];
                act_out[(size_t)(b0 + j0 + j) * ld_act + f] = f2bf(g / (1.f + __expf(-g)) * u);
              }
            }
          }
          asm volatile("bar.sync 2, 128;" ::: "memory");
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (EPI == kEpiClusterLL) {
    pdl_wait();  // (every thread: the pushes overwrite LL slots the predecessor chain consumed)
    const uint64_t tag =
        tag_epoch ? (uint64_t)((uint32_t)(*(volatile const uint64_t*)tag_epoch * tag_mult + tag_add)) << 32 : 0ull;
    cluster_ll_finish<BN>(reinterpret_cast<const float*>(smem), dst, tag,
                          (int)blockIdx.x / (int)cg::this_cluster().num_blocks(), N, B);
    cg::this_cluster().sync();
  }
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(Cfg::kTmemCols));
  }
  trace_mark(trs, 3);
  // fused allreduce: the last CTA to finish releases one arrival on every peer's counter
  signal_last_cta(sig);
}

// ------------------------------------------------------------------ host ---

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 tensor [rows][cols] with row pitch ld (elements), box [box_rows][64], SWIZZLE_128B.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                   int box_rows) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int64_t, int64_t, int>, CUtensorMap> cache;
  auto key = std::make_tuple(ptr, rows, cols, ld, box_rows);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *map = it->second;
    return kOk;
  }
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return fail(kCuda, "cuTensorMapEncodeTiled entry point unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * 2) % 16 != 0)
    return fail(kInvalid, "tensor map: base must be 16B aligned and row pitch a multiple of 16B");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  if (cache.size() > 4096) cache.clear();
  cache[key] = *map;
  return kOk;
}

static int pick_bn(int64_t b) {
  if (b <= 16) return 16;
  if (b <= 32) return 32;
  if (b <= 64) return 64;
  if (b <= 128) return 128;
  return 256;
}

// Split-K choice: minimise (waves x chunks-per-unit) for a 148-SM persistent grid,
// plus a small charge for the fp32 partial traffic the consumer has to reduce and
// one L2 round trip (~35 KB of one SM's weight stream) per 8 partials it sums.
int linear_splits(int64_t n, int64_t k, int64_t b) {
  const int bn = pick_bn(b);
  const int64_t tiles = ((n + kBM - 1) / kBM) * ((b + bn - 1) / bn);
  const int64_t chunks = (k + kBK - 1) / kBK;
  int best = 1;
  double best_cost = 1e30;
  const int max_s = (int)(chunks < 32 ? chunks : 32);
  for (int s = 1; s <= max_s; ++s) {
    const int64_t units = tiles * s;
    const int64_t waves = (units + kNumSMs - 1) / kNumSMs;
    const int64_t cpu = (chunks + s - 1) / s;
    const double weight_cost = (double)waves * (double)cpu * (kBM * kBK * 2);
    const double partial_cost = 0.25 * (double)s * (double)b * (double)n * 8.0 / kNumSMs;
    const double consumer_cost = (double)((s + 7) / 8) * 35.0 * 1024.0;
    const double cost = weight_cost + partial_cost + consumer_cost;
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

struct EpiArgs {
  DstList dst;
  long long split_stride;
  __nv_bfloat16* act_out;
  int ld_act;
  SignalSpec sig;
  const uint64_t* tag_epoch = nullptr;
  uint32_t tag_mult = 0;
  uint32_t tag_add = 0;
  ArgEpi arg{};
};

template <int BN, int EPI>
static int launch_gemm(const CUtensorMap& mw, const CUtensorMap& mx, const EpiArgs& e, int n, int b, int tiles,
                       int splits, int chunks, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  const int acts = (b + BN - 1) / BN;
  const int units = tiles * splits * acts;
  const int grid = units < kNumSMs ? units : kNumSMs;
  if constexpr (cluster_epi(EPI))  // one unit per CTA, the splits of a tile in one cluster
    return launch_kcs(gemm_swapab_kernel<BN, EPI>, dim3(units), dim3(kGemmThreads), splits, Cfg::kClusterSmemBytes,
                      stream, true, mw, mx, e.dst, e.split_stride, n, b, tiles, splits, chunks, acts, e.act_out,
                      e.ld_act, e.sig, e.tag_epoch, e.tag_mult, e.tag_add, e.arg);
  return launch_k(gemm_swapab_kernel<BN, EPI>, dim3(grid), dim3(kGemmThreads), Cfg::kSmemBytes, stream, true, mw,
                  mx, e.dst, e.split_stride, n, b, tiles, splits, chunks, acts, e.act_out, e.ld_act, e.sig,
                  e.tag_epoch, e.tag_mult, e.tag_add, e.arg);
}

template <int BN>
static int configure_one() {
  TPS_CUDA_TRY(cudaFuncSetAttribute(gemm_swapab_kernel<BN, kEpiPartial>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    GemmCfg<BN>::kSmemBytes));
  TPS_CUDA_TRY(cudaFuncSetAttribute(gemm_swapab_kernel<BN, kEpiSiluMul>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    GemmCfg<BN>::kSmemBytes));
  TPS_CUDA_TRY(cudaFuncSetAttribute(gemm_swapab_kernel<BN, kEpiArgmax>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    GemmCfg<BN>::kSmemBytes));
  TPS_MAX_CARVEOUT((gemm_swapab_kernel<BN, kEpiArgmax>));
  TPS_MAX_CARVEOUT((gemm_swapab_kernel<BN, kEpiPartial>));
  TPS_MAX_CARVEOUT((gemm_swapab_kernel<BN, kEpiSiluMul>));
  if constexpr (BN <= 64) {
    TPS_CUDA_TRY(cudaFuncSetAttribute(gemm_swapab_kernel<BN, kEpiClusterLL>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN>::kClusterSmemBytes));
    TPS_CUDA_TRY(cudaFuncSetAttribute(gemm_swapab_kernel<BN, kEpiClusterLL>,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TPS_MAX_CARVEOUT((gemm_swapab_kernel<BN, kEpiClusterLL>));
  }
  return kOk;
}

// Called from tps_init (never during stream capture).
int configure_gemm() {
  int rc = configure_one<16>();
  if (!rc) rc = configure_one<32>();
  if (!rc) rc = configure_one<64>();
  if (!rc) rc = configure_one<128>();
  if (!rc) rc = configure_one<256>();
  return rc;
}

// TPS_QKV_CLUSTER=<n>: largest split-K cluster of the cluster-reduced projection (default 8,
// the portable cluster size; 16 is allowed, 0 turns the cluster form off). (The name is
// round 1's, when the QKV projection had a cluster epilogue too.)
static int g_qkv_cluster = [] {
  const char* v = getenv("TPS_QKV_CLUSTER");
  return v ? atoi(v) : 8;
}();

// Split count of a cluster-reduced projection (tps_linear_push_ll_cluster), 0 when the shape
// does not take it: b <= 64 (one activation tile), every (tile, split) unit on its own SM
// (one wave), the splits of a tile within one cluster.
int cluster_splits(int64_t n, int64_t k, int64_t b) {
  if (g_qkv_cluster <= 0 || b < 1 || b > 64) return 0;
  const int64_t tiles = (n + kBM - 1) / kBM;
  const int64_t chunks = (k + kBK - 1) / kBK;
  if (tiles > kNumSMs) return 0;
  int s = linear_splits(n, k, b);
  int64_t cap = g_qkv_cluster < 16 ? g_qkv_cluster : 16;
  if (cap > chunks) cap = chunks;
  if (cap > kNumSMs / tiles) cap = kNumSMs / tiles;
  if (s > cap) s = cap;
  return s >= 1 ? s : 0;
}

template <int EPI>
static int dispatch(int bn, const CUtensorMap& mw, const CUtensorMap& mx, const EpiArgs& e, int n, int b, int tiles,
                    int splits, int chunks, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_gemm<16, EPI>(mw, mx, e, n, b, tiles, splits, chunks, st);
    case 32: return launch_gemm<32, EPI>(mw, mx, e, n, b, tiles, splits, chunks, st);
    case 64: return launch_gemm<64, EPI>(mw, mx, e, n, b, tiles, splits, chunks, st);
    case 128: return launch_gemm<128, EPI>(mw, mx, e, n, b, tiles, splits, chunks, st);
    default: return launch_gemm<256, EPI>(mw, mx, e, n, b, tiles, splits, chunks, st);
  }
}

static int prepare(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                   int64_t ldx, CUtensorMap* mw, CUtensorMap* mx, int* bn) {
  TPS_CHECK_ARG(w && x, "linear: null pointer");
  TPS_CHECK_ARG(n > 0 && k > 0 && b > 0 && b <= (1 << 20), "linear: need n,k > 0 and 1 <= b <= 2^20");
  TPS_CHECK_ARG(x_rows >= b && ldw >= k && ldx >= k, "linear: bad leading dimensions");
  *bn = pick_bn(b);
  int rc = make_tmap_bf16(mw, w, n, k, ldw, kBM);
  if (rc) return rc;
  return make_tmap_bf16(mx, x, x_rows, k, ldx, *bn);
}

int linear_push(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                int64_t ldx, const DstList& dst, int64_t split_stride, int splits, const SignalSpec& sig,
                cudaStream_t stream);

// out: fp32 split-K partials [splits][b][n] (the consumer sums them in split order).
int linear(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
           int64_t x_rows, int64_t ldx, float* out, int splits, cudaStream_t stream) {
  TPS_CHECK_ARG(out, "linear: null output");
  DstList dl;
  dl.n = 1;
  dl.p[0] = out;
  SignalSpec none;
  none.n = 0;
  none.done = nullptr;
  return linear_push(w, n, k, ldw, x, b, x_rows, ldx, dl, b * n, splits, none, stream);
}

// Partial of split s, row i, column j -> dst.p[d][s * split_stride + i * n + j] for every d,
// then (last CTA of the launch) +1 on every signal counter.
int linear_push(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                int64_t ldx, const DstList& dst, int64_t split_stride, int splits, const SignalSpec& sig,
                cudaStream_t stream) {
  const int64_t chunks = (k + kBK - 1) / kBK;
  TPS_CHECK_ARG(splits >= 1 && splits <= chunks, "linear: splits must be in [1, ceil(k/64)]");
  TPS_CHECK_ARG(dst.n >= 1 && dst.n <= kMaxPeers, "linear: 1..8 destinations");
  TPS_CHECK_ARG(split_stride >= b * n, "linear: split_stride must hold [b][n]");
  CUtensorMap mw, mx;
  int bn;
  int rc = prepare(w, n, k, ldw, x, b, x_rows, ldx, &mw, &mx, &bn);
  if (rc) return rc;
  EpiArgs e{dst, (long long)split_stride, nullptr, 0, sig};
  return dispatch<kEpiPartial>(bn, mw, mx, e, (int)n, (int)b, (int)((n + kBM - 1) / kBM), splits, (int)chunks,
                               stream);
}

// LL push: partial (split, i, j) -> dst.p[d][split * split_stride + i * n + j] as a uint64
// {fp32 bits, tag}, tag = (*tag_epoch) * tag_mult + tag_add (no counters, no signal).
int linear_push_ll(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                   int64_t ldx, const DstList& dst, int64_t split_stride, int splits, const uint64_t* tag_epoch,
                   uint32_t tag_mult, uint32_t tag_add, cudaStream_t stream) {
  const int64_t chunks = (k + kBK - 1) / kBK;
  TPS_CHECK_ARG(splits >= 1 && splits <= chunks, "linear: splits must be in [1, ceil(k/64)]");
  TPS_CHECK_ARG(dst.n >= 1 && dst.n <= kMaxPeers, "linear: 1..8 destinations");
  TPS_CHECK_ARG(split_stride >= b * n, "linear: split_stride must hold [b][n]");
  TPS_CHECK_ARG(tag_epoch != nullptr, "linear_push_ll: null epoch");
  for (int d = 0; d < dst.n; ++d)
    TPS_CHECK_ARG((reinterpret_cast<uintptr_t>(dst.p[d]) & 7) == 0, "linear_push_ll: destinations must be 8B aligned");
  CUtensorMap mw, mx;
  int bn;
  int rc = prepare(w, n, k, ldw, x, b, x_rows, ldx, &mw, &mx, &bn);
  if (rc) return rc;
  EpiArgs e{dst, (long long)split_stride, nullptr, 0, SignalSpec{}, tag_epoch, tag_mult, tag_add};
  e.sig.n = 0;
  return dispatch<kEpiPartial>(bn, mw, mx, e, (int)n, (int)b, (int)((n + kBM - 1) / kBM), splits, (int)chunks,
                               stream);
}

int linear_silu(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                int64_t ldx, void* act, int64_t ld_act, cudaStream_t stream) {
  TPS_CHECK_ARG(act && n % kBM == 0, "linear_silu: N = 2F must be a multiple of 128 (64-row gate/up blocks)");
  TPS_CHECK_ARG(ld_act >= n / 2, "linear_silu: ld_act must be >= F");
  const int64_t chunks = (k + kBK - 1) / kBK;
  CUtensorMap mw, mx;
  int bn;
  int rc = prepare(w, n, k, ldw, x, b, x_rows, ldx, &mw, &mx, &bn);
  if (rc) return rc;
  EpiArgs e{};
  e.dst.n = 0;
  e.act_out = reinterpret_cast<__nv_bfloat16*>(act);
  e.ld_act = (int)ld_act;
  e.sig.n = 0;
  return dispatch<kEpiSiluMul>(bn, mw, mx, e, (int)n, (int)b, (int)(n / kBM), 1, (int)chunks, stream);
}

// Row-parallel projection with the split-K reduction inside a cluster and one LL pair per
// element pushed to every destination at i * n + j (tag = (*tag_epoch) * tag_mult + tag_add).
int linear_push_ll_cluster(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b,
                           int64_t x_rows, int64_t ldx, const DstList& dst, const uint64_t* tag_epoch,
                           uint32_t tag_mult, uint32_t tag_add, cudaStream_t stream) {
  const int splits = cluster_splits(n, k, b);
  TPS_CHECK_ARG(splits >= 1, "linear_push_ll_cluster: shape not supported (see tps_cluster_splits)");
  TPS_CHECK_ARG(dst.n >= 1 && dst.n <= kMaxPeers && tag_epoch, "linear_push_ll_cluster: 1..8 destinations, epoch");
  for (int d = 0; d < dst.n; ++d)
    TPS_CHECK_ARG((reinterpret_cast<uintptr_t>(dst.p[d]) & 7) == 0, "linear_push_ll_cluster: 8B-aligned slots");
  const int64_t chunks = (k + kBK - 1) / kBK;
  CUtensorMap mw, mx;
  int bn;
  int rc = prepare(w, n, k, ldw, x, b, x_rows, ldx, &mw, &mx, &bn);
  if (rc) return rc;
  EpiArgs e{dst, 0, nullptr, 0, SignalSpec{}, tag_epoch, tag_mult, tag_add};
  e.sig.n = 0;
  const int tiles = (int)((n + kBM - 1) / kBM);
  switch (bn) {
    case 16: return launch_gemm<16, kEpiClusterLL>(mw, mx, e, (int)n, (int)b, tiles, splits, (int)chunks, stream);
    case 32: return launch_gemm<32, kEpiClusterLL>(mw, mx, e, (int)n, (int)b, tiles, splits, (int)chunks, stream);
    default: return launch_gemm<64, kEpiClusterLL>(mw, mx, e, (int)n, (int)b, tiles, splits, (int)chunks, stream);
  }
}

// LM head with the greedy argmax stage in the epilogue: logits [b][n] fp32 (splits = 1) and
// cand[i][t] = {max, smallest index on ties} over columns [128 t, 128 t + 128) (+ vocab0).
int linear_argmax(const void* w, int64_t n, int64_t k, int64_t ldw, const void* x, int64_t b, int64_t x_rows,
                  int64_t ldx, float* logits, void* cand, int vocab0, cudaStream_t stream) {
  TPS_CHECK_ARG(logits && cand, "linear_argmax: null output");
  const int64_t chunks = (k + kBK - 1) / kBK;
  CUtensorMap mw, mx;
  int bn;
  int rc = prepare(w, n, k, ldw, x, b, x_rows, ldx, &mw, &mx, &bn);
  if (rc) return rc;
  EpiArgs e{};
  e.dst.n = 1;
  e.dst.p[0] = logits;
  e.split_stride = b * n;
  e.sig.n = 0;
  const int tiles = (int)((n + kBM - 1) / kBM);
  e.arg = ArgEpi{reinterpret_cast<ArgmaxCand*>(cand), tiles, vocab0};
  return dispatch<kEpiArgmax>(bn, mw, mx, e, (int)n, (int)b, tiles, 1, (int)chunks, stream);
}

int trace_register_gemm(uint64_t* p, unsigned int* c, unsigned int n) { return trace_register(p, c, n); }

}  // namespace tps
