// Shared device/host definitions of libvoxmap_b200 (sm_100a).
//
// Exactness: every translation unit is compiled with --fmad=false and IEEE
// division/sqrt, and the FP64 geometry below spells out the association
// order pinned by oracle/eigen_shim (3-term sums a0 + (a1 + a2)), so the
// GPU reproduces the reference's voxel centres, transforms and projections
// bit-for-bit (SURVEY.md §8(a) "exact-arithmetic contract").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "voxmap_b200.h"

namespace vxm {

constexpr int kVPS = 8;    // kVoxelsPerSide  (core/indexing.hpp:28)
constexpr int kVPB = 512;  // kVoxelsPerBlock (core/indexing.hpp:29-30)

// ---- packed block keys ------------------------------------------------------
// GridIndex -> 63-bit key, 21 bits per axis with a +2^20 bias, x most
// significant: unsigned key order == lexicographic GridIndex order
// (operator<=> indexing.hpp:38).  Coordinates must lie in [-2^20+2, 2^20-3]
// so that composed +-1 neighbour shifts stay representable.
constexpr int kKeyBits = 21;
constexpr int64_t kKeyBias = int64_t(1) << 20;
constexpr uint64_t kKeyMask = (uint64_t(1) << kKeyBits) - 1;
constexpr uint64_t kEmptyKey = ~uint64_t(0);
constexpr int32_t kCoordMin = -(1 << 20) + 2;
constexpr int32_t kCoordMax = (1 << 20) - 3;

__host__ __device__ inline uint64_t pack_key(int32_t x, int32_t y, int32_t z) {
  return (uint64_t(int64_t(x) + kKeyBias) << (2 * kKeyBits)) |
         (uint64_t(int64_t(y) + kKeyBias) << kKeyBits) | uint64_t(int64_t(z) + kKeyBias);
}
__host__ __device__ inline int32_t key_x(uint64_t k) {
  return int32_t(int64_t((k >> (2 * kKeyBits)) & kKeyMask) - kKeyBias);
}
__host__ __device__ inline int32_t key_y(uint64_t k) {
  return int32_t(int64_t((k >> kKeyBits) & kKeyMask) - kKeyBias);
}
__host__ __device__ inline int32_t key_z(uint64_t k) {
  return int32_t(int64_t(k & kKeyMask) - kKeyBias);
}
// Shift one axis by s (=+-1) without unpacking: fields are biased, so adding
// s << shift never borrows across fields for in-range coordinates.
__host__ __device__ inline uint64_t key_shift(uint64_t k, int axis, int s) {
  const int sh = axis == 0 ? 2 * kKeyBits : (axis == 1 ? kKeyBits : 0);
  return s > 0 ? k + (uint64_t(1) << sh) : k - (uint64_t(1) << sh);
}
__host__ __device__ inline bool coord_ok(int64_t c) { return c >= kCoordMin && c <= kCoordMax; }

// ---- open-addressing block hash (key -> pool slot) ---------------------------
__host__ __device__ inline uint32_t hash_key(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return uint32_t(k);
}

struct HashView {
  uint64_t* keys;
  int32_t* vals;
  uint32_t mask;
};

// Probing is bounded by the table size (tables are kept at most half full, so
// the bound is never reached; it only turns a corrupted table into a miss
// instead of a GPU hang).
__device__ inline int32_t hash_find(const HashView& h, uint64_t k) {
  uint32_t i = hash_key(k) & h.mask;
  for (uint32_t n = 0; n <= h.mask; ++n) {
    const uint64_t kk = __ldg(h.keys + i);
    if (kk == k) return __ldg(h.vals + i);
    if (kk == kEmptyKey) return -1;
    i = (i + 1) & h.mask;
  }
  return -1;
}
// Mutable-table lookup (no read-only cache): used in kernels that also insert.
__device__ inline int32_t hash_find_rw(const HashView& h, uint64_t k) {
  uint32_t i = hash_key(k) & h.mask;
  for (uint32_t n = 0; n <= h.mask; ++n) {
    const uint64_t kk = h.keys[i];
    if (kk == k) return h.vals[i];
    if (kk == kEmptyKey) return -1;
    i = (i + 1) & h.mask;
  }
  return -1;
}
// Keys inserted by one launch are unique, so CAS-claim then write the value.
__device__ inline void hash_insert(const HashView& h, uint64_t k, int32_t v) {
  uint32_t i = hash_key(k) & h.mask;
  for (uint32_t n = 0; n <= h.mask; ++n) {
    const unsigned long long prev =
        atomicCAS(reinterpret_cast<unsigned long long*>(h.keys + i),
                  (unsigned long long)kEmptyKey, (unsigned long long)k);
    if (prev == kEmptyKey || prev == k) {
      h.vals[i] = v;
      return;
    }
    i = (i + 1) & h.mask;
  }
}

// ---- per-layer device metadata ------------------------------------------------
struct LayerMeta {
  uint32_t num_blocks;   // allocated blocks (slots [0, num_blocks) are live)
  uint32_t cur;          // ESDF: which of the two pools holds the current field
  uint32_t round_epoch;  // ESDF: monotone round counter for dirty stamps
  uint32_t pad;
};

// Per-context status written by kernels, read by the host after a sync.
struct DevStatus {
  uint32_t pool_overflow;    // physical pool too small: host grows and re-runs
  uint32_t capacity_error;   // Layer::max_blocks exceeded (MapCapacityError)
  uint32_t bitmap_overflow;  // ray left the candidate cube (internal error)
  uint32_t n_candidates;
  uint32_t n_new;
  uint32_t n_changed;
  uint32_t n_effective;
  uint32_t n_esdf_new;
  uint32_t any_update;       // mark: some block queued to update/clear
  uint32_t rounds;           // lowering rounds of the last lower
  uint32_t n_out;            // generic output count
  uint32_t n_aux;            // generic aux count
  // work counters (algorithmic-bytes model)
  uint32_t vox_read;         // integrate: existing voxels read
  uint32_t vox_upd;          // integrate: voxels written
  uint32_t sum_dirty;        // lower: dirty blocks summed over rounds >= 2
  uint32_t sum_pairs;        // lower: face pairs exchanged
  uint32_t cmp_blocks;       // lower: blocks compared for the changed set
  uint32_t n_esdf_blocks;    // ESDF blocks after the update
  uint32_t meta_blocks;      // copy of the layer's LayerMeta {num_blocks, cur}
  uint32_t meta_cur;         //   taken with the status read (one sync per call)
  uint32_t watchdog;         // a bounded dependency wait expired (internal error)
  uint32_t pad3[3];
  uint32_t meta2_blocks;     // second layer's meta (fused frame update: TSDF + ESDF)
  uint32_t meta2_cur;
  uint32_t integ_claim;      // k_integrate: candidate blocks claimed (dynamic schedule)
  uint32_t quiet_blocks;     // lower: round-1 blocks skipped by the quiet chain (no read, no copy)
};

// ---- decoupled look-back scan over (a, b) count pairs ------------------------
// Tile status: [63:62] flag (1 aggregate, 2 inclusive prefix), [61:31] a, [30:0] b.
struct ScanTiles {
  unsigned long long* status;  // >= num_tiles entries, zero before use
  unsigned long long* next;    // the other status buffer; cleared by this pass
  uint32_t* ticket;            // this pass's tile ticket counter (zero before use)
  uint32_t* next_ticket;       // the next pass's counter; reset by this pass
  uint32_t n_next;             // entries of `next` to clear
};

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
__device__ inline unsigned long long pack_ab(uint32_t a, uint32_t b) {
  return (unsigned long long)(a & 0x7fffffffu) << 31 | (b & 0x7fffffffu);
}
__device__ inline uint32_t unpack_a(unsigned long long v) { return uint32_t(v >> 31) & 0x7fffffffu; }
__device__ inline uint32_t unpack_b(unsigned long long v) { return uint32_t(v) & 0x7fffffffu; }

// ---- misc --------------------------------------------------------------------
// Programmatic dependent launch (PDL): the kernels of the per-frame chain are
// launched with programmatic stream serialization (launch_pdl), so a kernel's
// CTAs are dispatched while its predecessor drains.  Every such kernel calls
// pdl_wait() before touching memory (it returns once the predecessor has
// completed and flushed) and pdl_trigger() to let its own successor launch.
// Both are no-ops in a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#define VXM_CUDA(call)                                                             \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      throw ::vxm::Error(VXM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline uint32_t ceil_div(uint64_t a, uint64_t b) { return uint32_t((a + b - 1) / b); }

}  // namespace vxm
