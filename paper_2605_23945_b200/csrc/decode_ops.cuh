// Parameter structs shared by the decode kernels and the C-ABI layer.
#pragma once
#include <stdint.h>

namespace tps {

constexpr int kMaxSrc = 64;
constexpr int kMaxPeers = 8;

// An ordered list of fp32 [rows][cols] partial buffers to be summed
// (split-K partials of one rank, or one slot per TP rank). Summation order
// is the list order, so every rank of a TP group reduces bitwise-identically.
struct SrcList {
  const float* p[kMaxSrc];
  int n;
};

// Cross-GPU completion counter wait: spin until *ctr >= (*epoch) * mult + add
// (or >= add when epoch is null). Counters only grow, so CUDA-graph replays
// need no host-side reset.
struct WaitSpec {
  const uint64_t* ctr;
  const uint64_t* epoch;
  uint64_t mult;
  uint64_t add;
};

// After a CTA's stores are globally visible, add 1 to each listed counter
// (local or NVLink-peer), with release semantics at system scope.
// The last CTA of the launch (detected with the per-launch-site `done` counter,
// which it resets) issues the signals, so each rank contributes exactly one
// arrival per phase regardless of grid size / batch bucket.
struct SignalSpec {
  uint64_t* ctr[kMaxPeers];
  int n;
  unsigned int* done;
};

// Destination list for a reduce-and-push: the same [rows][cols] fp32 result is
// stored to every listed buffer (this rank's slot in each peer's receive area).
struct DstList {
  float* p[kMaxPeers];
  int n;
};

struct ArgmaxCand {
  float val;
  int idx;
};

struct CandList {
  const ArgmaxCand* p[kMaxPeers];
  int n;
};

}  // namespace tps
