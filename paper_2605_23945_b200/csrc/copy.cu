// Switch Executor data movement: batched peer pulls for weight reshard and
// KV-page migration, plus the device barrier and CUDA-IPC plumbing.
//
// Replaces the layer-wise All-Gather + Slice the reference plans
// (plan_weight_reshard / plan_kv_migration, tpshift/reshard.py:80-151) with
// one-sided pulls: every target rank reads exactly the canonical slices it
// owns from whichever rank holds them (local HBM when the slice is already
// resident, an NVLink peer otherwise). Copies are byte-exact by construction.
//
// Work items are 1-D contiguous chunks (host-side planner splits 2-D slices
// into rows / <=64 KB pieces). Two engines:
//   mode 0: LSU copy, 4 x 16 B loads in flight per thread, persistent grid;
//   mode 1: TMA-staged copy, cp.async.bulk global->smem->global through a
//           2-deep ring of 48 KB buffers per CTA, 2 CTAs per SM (no register round trip).
#include "common.cuh"

namespace tps {

struct CopyItem {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t bytes;
  uint64_t reserved;
};

constexpr int kCopyThreads = 256;

__global__ void __launch_bounds__(kCopyThreads) copy_items_lsu_kernel(const CopyItem* __restrict__ items,
                                                                      int n) {
  for (int it = blockIdx.x; it < n; it += gridDim.x) {
    const CopyItem ci = items[it];
    const bool aligned = ((reinterpret_cast<uintptr_t>(ci.src) | reinterpret_cast<uintptr_t>(ci.dst)) & 15u) == 0;
    const uint64_t nvec = aligned ? ci.bytes / 16 : 0;
    const int4* s = reinterpret_cast<const int4*>(ci.src);
    int4* d = reinterpret_cast<int4*>(ci.dst);
    uint64_t i = threadIdx.x;
    for (; i + 3 * kCopyThreads < nvec; i += 4 * kCopyThreads) {
      int4 v0 = s[i], v1 = s[i + kCopyThreads], v2 = s[i + 2 * kCopyThreads], v3 = s[i + 3 * kCopyThreads];
      d[i] = v0;
      d[i + kCopyThreads] = v1;
      d[i + 2 * kCopyThreads] = v2;
      d[i + 3 * kCopyThreads] = v3;
    }
    for (; i < nvec; i += kCopyThreads) d[i] = s[i];
    for (uint64_t j = nvec * 16 + threadIdx.x; j < ci.bytes; j += kCopyThreads) ci.dst[j] = ci.src[j];
  }
}

constexpr int kBulkMaxDepth = 8;
// ring geometry (TPS_COPY_BUF_KB x TPS_COPY_DEPTH per CTA, TPS_COPY_CTAS_PER_SM CTAs per SM).
// Swept on the config-5 switch microbench (Qwen2.5-7B TP1 -> TP2, 16 samples at 4K, 20.1 GB of
// items): 32 KB x 4 x 2 (one CTA resident per SM) 2465 GB/s; 32 x 2 x 3 2848-2881; 16 x 2 x 4
// 2862; 48 x 2 x 2 2968 (91 % of the read+write copy peak) -- two 96 KB CTAs per SM.
static int g_bulk_buf = [] {
  const char* v = getenv("TPS_COPY_BUF_KB");
  return (v ? atoi(v) : 48) * 1024;
}();
static int g_bulk_depth = [] {
  const char* v = getenv("TPS_COPY_DEPTH");
  const int d = v ? atoi(v) : 2;
  return d < 2 ? 2 : (d > kBulkMaxDepth ? kBulkMaxDepth : d);
}();
static int g_bulk_ctas = [] {
  const char* v = getenv("TPS_COPY_CTAS_PER_SM");
  return v ? atoi(v) : 2;
}();

// One elected thread per CTA drives a depth-deep ring: loads of chunks
// k+1..k+depth-1 are in flight while chunk k is being stored.
__global__ void __launch_bounds__(32) copy_items_tma_kernel(const CopyItem* __restrict__ items, int n,
                                                            int kBulkBuf, int kBulkDepth) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ __align__(8) uint64_t bars[kBulkMaxDepth];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kBulkDepth; ++i) mbar_init(&bars[i], 1);
  fence_barrier_init();
  int git = blockIdx.x;
  uint64_t goff = 0;
  auto next = [&](const uint8_t*& s, uint8_t*& d, uint32_t& len) -> bool {
    while (git < n) {
      const CopyItem ci = items[git];
      if (((reinterpret_cast<uintptr_t>(ci.src) | reinterpret_cast<uintptr_t>(ci.dst) | ci.bytes) & 15u) != 0) {
        // not bulk-copyable (the host routes such items to the LSU engine): plain bytes
        for (uint64_t j = goff; j < ci.bytes; ++j) ci.dst[j] = ci.src[j];
        git += gridDim.x;
        goff = 0;
        continue;
      }
      if (goff < ci.bytes) {
        const uint64_t rem = ci.bytes - goff;
        len = (uint32_t)(rem < (uint64_t)kBulkBuf ? rem : (uint64_t)kBulkBuf);
        s = ci.src + goff;
        d = ci.dst + goff;
        goff += len;
        return true;
      }
      git += gridDim.x;
      goff = 0;
    }
    return false;
  };
  uint8_t* dsts[kBulkMaxDepth];
  uint32_t lens[kBulkMaxDepth];
  uint32_t phases = 0;
  int head = 0, tail = 0;
  const uint8_t* s;
  uint8_t* d;
  uint32_t len;
  while (tail < kBulkDepth && next(s, d, len)) {
    const int sl = tail % kBulkDepth;
    mbar_arrive_expect_tx(&bars[sl], len);
    bulk_g2s(sbuf + sl * kBulkBuf, s, len, &bars[sl]);
    dsts[sl] = d;
    lens[sl] = len;
    ++tail;
  }
  while (head < tail) {
    const int sl = head % kBulkDepth;
    mbar_wait(&bars[sl], (phases >> sl) & 1u);
    phases ^= (1u << sl);
    bulk_s2g(dsts[sl], sbuf + sl * kBulkBuf, lens[sl]);
    bulk_commit();
    ++head;
    if (next(s, d, len)) {
      bulk_wait_read<0>();  // the store just issued has read its smem slot
      const int sl2 = tail % kBulkDepth;
      mbar_arrive_expect_tx(&bars[sl2], len);
      bulk_g2s(sbuf + sl2 * kBulkBuf, s, len, &bars[sl2]);
      dsts[sl2] = d;
      lens[sl2] = len;
      ++tail;
    }
  }
  bulk_wait<0>();
}

int configure_copy() {
  TPS_CUDA_TRY(cudaFuncSetAttribute(copy_items_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    g_bulk_buf * g_bulk_depth));
  return kOk;
}

int copy_items(const void* items, int n, int mode, int grid, cudaStream_t st) {
  TPS_CHECK_ARG(n >= 0, "copy_items: n >= 0");
  if (n == 0) return kOk;
  if (grid <= 0) grid = (mode == 1 ? g_bulk_ctas : 2) * kNumSMs;
  if (grid > n) grid = n;
  if (mode == 0) {
    copy_items_lsu_kernel<<<grid, kCopyThreads, 0, st>>>(reinterpret_cast<const CopyItem*>(items), n);
  } else if (mode == 1) {
    const int smem = g_bulk_buf * g_bulk_depth;
    copy_items_tma_kernel<<<grid, 32, smem, st>>>(reinterpret_cast<const CopyItem*>(items), n, g_bulk_buf,
                                                  g_bulk_depth);
  } else {
    return fail(kInvalid, "copy_items: mode must be 0 (LSU) or 1 (TMA bulk)");
  }
  TPS_LAUNCH_CHECK();
  return kOk;
}

// ----------------------------------------------- KV-page migration items ----
// The Switch Executor's KV plan, expanded on the device from page tables.
// One move = one migrating sample x one run of kv heads that are contiguous in
// both pools and come from one source rank. Its items are the (layer, k|v,
// valid page) triples: every one is a single contiguous n_heads x 16 KB range
// in both pool layouts [L][2][pages][n_kv][64][D] (kv head is the fastest index
// above the page's tokens), so the host ships O(samples) descriptors instead of
// O(samples x layers x pages) copy items (tpshift/reshard.py:113-151).
struct KVMove {
  const uint8_t* src_kv;
  const int32_t* src_pages;
  const int32_t* dst_pages;
  int32_t src_num_pages, src_nkv, src_head;
  int32_t dst_head, n_heads, n_pages;
  int64_t first_item;
};
static_assert(sizeof(KVMove) == 56, "tps_kv_move layout");

__global__ void __launch_bounds__(256) kv_move_items_kernel(const KVMove* __restrict__ moves, int n_moves,
                                                            int64_t n_items, uint8_t* dst_kv, int dst_num_pages,
                                                            int dst_nkv, int64_t chunk, CopyItem* __restrict__ out,
                                                            int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_items;
       i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_moves - 1;  // last move with first_item <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (moves[mid].first_item <= i) lo = mid; else hi = mid - 1;
    }
    const KVMove& m = moves[lo];
    const int64_t j = i - m.first_item;
    const int p = (int)(j % m.n_pages);
    const int64_t lkv = j / m.n_pages;  // layer * 2 + (0: K, 1: V)
    const int sp = m.src_pages[p], dp = m.dst_pages[p];
    CopyItem it;
    if (sp < 0 || sp >= m.src_num_pages || dp < 0 || dp >= dst_num_pages || m.src_head + m.n_heads > m.src_nkv ||
        m.dst_head + m.n_heads > dst_nkv) {
      if (bad) atomicAdd(bad, 1);
      it.src = nullptr; it.dst = nullptr; it.bytes = 0; it.reserved = 0;  // copies nothing
    } else {
      it.src = m.src_kv + ((lkv * m.src_num_pages + sp) * m.src_nkv + m.src_head) * chunk;
      it.dst = dst_kv + ((lkv * dst_num_pages + dp) * dst_nkv + m.dst_head) * chunk;
      it.bytes = (uint64_t)m.n_heads * chunk;
      it.reserved = 0;
    }
    out[i] = it;
  }
}

int kv_move_items(const void* moves, int n_moves, int64_t n_items, void* dst_kv, int dst_num_pages, int dst_nkv,
                  int64_t chunk_bytes, void* items_out, int* bad, cudaStream_t st) {
  TPS_CHECK_ARG(n_moves >= 0 && n_items >= 0 && chunk_bytes > 0 && (chunk_bytes & 15) == 0,
                "kv_move_items: bad sizes");
  if (n_items == 0) return kOk;
  TPS_CHECK_ARG(moves && dst_kv && items_out && n_moves > 0, "kv_move_items: null argument");
  int64_t blocks = (n_items + 255) / 256;
  if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
  kv_move_items_kernel<<<(int)blocks, 256, 0, st>>>(reinterpret_cast<const KVMove*>(moves), n_moves, n_items,
                                                     reinterpret_cast<uint8_t*>(dst_kv), dst_num_pages, dst_nkv,
                                                     chunk_bytes, reinterpret_cast<CopyItem*>(items_out), bad);
  TPS_LAUNCH_CHECK();
  return kOk;
}

// ------------------------------------------------------ device barrier ----
// Epoch barrier with one slot per source rank: rank q stores the barrier's epoch
// into slot q of every peer's slot array (plain 8-B stores: idempotent, a replayed or
// duplicated signal cannot over-count), then waits until every peer's slot in its own
// array holds >= epoch. Replaces round 1's shared counter of relaxed atomic adds, whose
// lazily queued zero-fill could wipe a fast peer's early add and hang the barrier (a wiped
// epoch store is superseded by the next barrier's; tests/test_barrier_protocol.py).
constexpr int kMaxPeerArgs = 16;
struct PeerPtrs {
  uint64_t* p[kMaxPeerArgs];
};

__global__ void barrier_kernel_v(PeerPtrs peers, int npeers, const uint64_t* my_slots, int nslots, int self_slot,
                                 uint64_t epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();  // everything this stream wrote before the barrier is visible first
  for (int i = 0; i < npeers; ++i) st_relaxed_sys_u64(peers.p[i], epoch);
  for (int j = 0; j < nslots; ++j)
    if (j != self_slot) wait_counter_geq(my_slots + j, epoch);
  __threadfence_system();
}

int barrier(uint64_t* const* peer_slots, int npeers, const uint64_t* my_slots, int nslots, int self_slot,
            uint64_t epoch, cudaStream_t st) {
  TPS_CHECK_ARG(npeers >= 0 && npeers <= kMaxPeerArgs && my_slots && nslots >= 0 && nslots <= kMaxPeerArgs + 1,
                "barrier: bad args");
  PeerPtrs pp{};
  for (int i = 0; i < npeers; ++i) pp.p[i] = peer_slots[i];
  barrier_kernel_v<<<1, 32, 0, st>>>(pp, npeers, my_slots, nslots, self_slot, epoch);
  TPS_LAUNCH_CHECK();
  return kOk;
}

// ------------------------------------------------------------------ IPC ---
typedef CUresult (*GetAddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

int ipc_get_handle(const void* ptr, void* handle_out, int64_t* offset_out) {
  TPS_CHECK_ARG(ptr && handle_out && offset_out, "ipc_get_handle: null argument");
  static GetAddrRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(kCuda, "cuMemGetAddressRange entry point unavailable");
    fn = reinterpret_cast<GetAddrRangeFn>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(kCuda, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  TPS_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - (uintptr_t)base);
  return kOk;
}

int ipc_open(const void* handle, void** base_out) {
  TPS_CHECK_ARG(handle && base_out, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  TPS_CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return kOk;
}

int ipc_close(void* base) {
  TPS_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return kOk;
}

}  // namespace tps
