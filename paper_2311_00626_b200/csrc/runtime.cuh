// Host-side runtime of libvoxmap_b200: contexts, layers (device block pool +
// open-addressing hash), block lists, scratch management.  Kernels live in
// view.cu / integrate.cu / esdf.cu / query.cu; the C-ABI in capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace vxm {

// Growable device allocation (contents are NOT preserved on growth).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void ensure(size_t n);
  void release();
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// Double-buffered decoupled-look-back scan state (see common.cuh ScanTiles).
struct ScanState {
  unsigned long long* status[2] = {nullptr, nullptr};
  uint32_t* tickets = nullptr;  // [2]
  uint32_t cap = 0;             // entries per status buffer
  int parity = 0;
};

struct Context {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  DevStatus* d_status = nullptr;
  DevStatus* h_status = nullptr;      // pinned, mapped: written by k_status_out
  DevStatus* h_status_dev = nullptr;  // its device address
  uint64_t launches = 0;
  ScanState scan;
  uint32_t call_epoch = 0;
  // sharding: owner(g) = floor(g.x / slab) mod world
  int rank = 0, world = 1, slab = 16;
  // scratch
  DevBuf depth;           // staged depth image
  DevBuf bitmap[2];       // touched-cell bitmaps (candidate cube), alternating by call:
  int bitmap_parity = 0;  //   the call on one clears the other for the next call
  uint64_t bitmap_clean[2] = {0, 0};  // words known zero in each
  DevBuf cand_keys;       // uint64 candidate keys (sorted)
  DevBuf cand_slots;      // int32 slot | new flag
  DevBuf cand_flags;      // uint8 per candidate (changed)
  DevBuf lidar_dirs;      // double3 per LiDAR pixel (host glibc LUT)
  DevBuf atan_tab;        // double4 x kAtanTabN: the LiDAR projection's atan2 table (integrate.cu)
  vxm_lidar lut_key{};
  bool lut_valid = false;
  DevBuf cam_dirs;        // double2 per camera tile: ((u - cu) / fu, (v - cv) / fv)
  vxm_camera cam_key{};
  int cam_key_w = 0, cam_key_h = 0, cam_key_tile = 0;
  bool cam_lut_valid = false;
  DevBuf tmp[6];          // ESDF / list scratch
  DevBuf lower_cta;       // k_lower_xr: per-CTA counts of the changed-list compaction
  DevBuf cub_tmp;

  // work counters and optional per-kernel event timing
  vxm_stats stats{};
  bool profile = false;
  struct Pending {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> spare_events;
  std::map<std::string, std::pair<double, uint64_t>> ktime;
  const char* prof_name = nullptr;
  cudaEvent_t prof_a = nullptr;
  struct BlockList* scratch_in = nullptr;  // reused host-input list (C-ABI host paths)
  // The changed list the last host-buffer integrate returned (device keys +
  // host copy): an update_esdf on an identical host list reuses its device keys
  // instead of uploading them again.  Cleared by the list's destructor.
  struct BlockList* last_host_out = nullptr;
  // Deferred mode (fused frame update): drivers enqueue their work and leave
  // the status read, error checks and meta adoption to the caller's one sync.
  bool deferred = false;

  // Launch geometry per kernel on THIS context's device (resident CTAs per
  // SM; one-time function attributes).  Keyed by context, not process-wide:
  // contexts on different devices (or threads) never share a stale entry.
  std::mutex geo_mu;
  std::map<const void*, int> resident;
  std::set<const void*> attr_done;
  int resident_per_sm(const void* kernel, int threads, size_t smem = 0, int cap = 1 << 30);
  // runs `set` once per kernel on this context (cudaFuncSetAttribute etc.)
  template <typename F>
  void once_attr(const void* kernel, F&& set) {
    std::lock_guard<std::mutex> g(geo_mu);
    if (attr_done.insert(kernel).second) set();
  }

  // Scan pass bookkeeping: returns the ScanTiles for the next pass with at
  // most `tiles` tiles, clearing the other buffer for the pass after.
  ScanTiles next_scan(uint32_t tiles);
  void count_launch(int n = 1) { launches += uint64_t(n); }
  // flush the queued status copies, copy status to the host, sync; with
  // `last` (the call's final read) the same kernel zeroes the device status,
  // so the next call's reset_status needs no memset
  void sync_status(bool last = false);
  bool status_zero = false;  // the device status is known to be zero
  // the device status for a kernel that writes it (no longer known zero)
  DevStatus* status_w() {
    status_zero = false;
    return d_status;
  }
  // Small device-to-device word copies into the status (counts, metas) are
  // queued and done by ONE kernel before the status read, instead of one
  // cudaMemcpyAsync each (each is a separate stream operation).
  struct WordCopy {
    const uint32_t* src;
    uint32_t* dst;
  };
  std::vector<WordCopy> status_copies;
  // A host-bound list's unpack (BlockList::enqueue_host), deferred into the
  // status-out kernel of the next sync_status: one launch fewer per host call.
  struct EmitHost {
    const uint64_t* keys = nullptr;
    const uint32_t* n_ptr = nullptr;
    vxm_grid_index* out = nullptr;
    uint32_t* out_n = nullptr;
    uint32_t cap = 0;
    uint32_t grid = 0;  // 0: none pending
    const void* list = nullptr;
  };
  EmitHost emit;
  void flush_emit();  // launches a pending unpack on its own
  void queue_copy(const uint32_t* src, uint32_t* dst, int n_words = 1) {
    for (int i = 0; i < n_words; ++i) status_copies.push_back({src + i, dst + i});
  }
  void flush_copies();
  void reset_status();
  void prof_begin(const char* name);
  void prof_end();
  void prof_resolve();  // after a stream sync
};

// Cross-round ring counters (lower_xr.cu): 17 counters, one 256-byte line
// each, after 64 words of list / work counters in Layer::dirty_count.
constexpr int kRingStride = 64;
constexpr int kRingOffset = 64;
constexpr int kDirtyCountWords = kRingOffset + 17 * kRingStride;

struct Layer {
  Context* ctx = nullptr;
  int type = VXM_LAYER_TSDF;
  double vs = 0.0;
  uint64_t max_blocks = 0;
  uint32_t capacity = 0;        // pool slots
  uint32_t num_blocks = 0;      // host mirror, exact after each synchronous call
  HashView hash{nullptr, nullptr, 0};
  uint32_t hash_cap = 0;
  uint64_t* slot_keys = nullptr;  // slot -> key
  void* pool[2] = {nullptr, nullptr};
  LayerMeta* meta = nullptr;    // device
  uint32_t cur_host = 0;        // host mirror of meta->cur (ESDF)
  // ESDF-only
  int32_t* nbr = nullptr;                  // [cap][6] neighbour slots (+x,-x,+y,-y,+z,-z)
  uint64_t* sorted_keys[2] = {nullptr, nullptr};
  int32_t* sorted_slots[2] = {nullptr, nullptr};
  int sorted_parity = 0;
  uint32_t* stamp_dirty[2] = {nullptr, nullptr};
  uint32_t* stamp_mark = nullptr;   // call epoch when mark changed the block
  uint32_t* stamp_new = nullptr;    // call epoch when the block was allocated
  uint32_t* stamp_lchg = nullptr;   // round epoch of the last lowering change
  int32_t* dirty_list[2] = {nullptr, nullptr};
  uint32_t* dirty_count = nullptr;  // [kDirtyCountWords]: list counts, work counters, round-1
                                    // split counters; from kRingOffset the cross-round ring
  unsigned long long* dlist[2] = {nullptr, nullptr};  // [cap] (epoch << 32 | slot) dirty lists
  unsigned long long* pair_face[3] = {nullptr, nullptr, nullptr};  // [cap][2] faces a pair changed
  unsigned long long* line_mask = nullptr;  // [cap][3] lines changed by border phases
  uint32_t* stamp_swept = nullptr;          // round epoch of the block's last sweep
  uint8_t* site_any = nullptr;              // 0: the block holds no site (exact or conservative 1)
  uint8_t* site_near = nullptr;             // k_lower_xr scratch: sites near the block (per launch)
  int32_t* r1_list = nullptr;               // k_lower_xr scratch: [3][cap] round-1 pair lists
  uint32_t* stamp_pair[3] = {nullptr, nullptr, nullptr};  // round epoch of pair (b, b+axis)
  uint32_t* stamp_r1same = nullptr;  // call epoch: round 1 left the block byte-identical
  uint32_t* stamp_quiet = nullptr;   // call epoch: both pools hold the block and reset is its identity
  // The quiet chain (k_lower_xr): a block an update left untouched, whose
  // round-1 reset was the identity, has the same bytes in both pools, so the
  // next update's round 1 need neither read nor copy it — as long as nothing
  // else wrote the layer in between.  esdf_gen counts every writer of ESDF
  // blocks (mark, lowering, clear, growth, user writes, shards); the chain
  // holds while it equals xr_gen, its value right after the last k_lower_xr
  // update (epoch xr_epoch, limits xr_max_sq / xr_cap_sq).
  uint64_t esdf_gen = 0, xr_gen = ~uint64_t(0);
  uint32_t xr_epoch = 0;
  uint32_t xr_quiet = 0;  // blocks the last update's round 1 found quiet
  // Mark skip, on one process-wide clock (next_mod_tick): a source layer
  // stamps every block an integrate changed (stamp_mod; a host write of its
  // blocks raises mod_floor over all earlier stamps), an ESDF block the tick
  // of its last marking (mark_stamp).  A block whose TSDF source block is
  // unchanged since then re-marks to the same bytes (mark_sites is voxel-local
  // for a TSDF source, and only marking writes the flags), so k_mark skips it
  // — while the quiet chain holds and the source and site threshold are those
  // of the last update (else mark_floor invalidates every stamp).
  uint32_t* stamp_mod = nullptr;   // source layers: [cap] tick of the block's last change
  uint32_t mod_floor = 0;
  uint32_t* mark_stamp = nullptr;  // ESDF: [cap] tick of the block's last marking
  uint32_t mark_floor = 0;
  bool mark_chain = false;         // ESDF: this update may trust the stamps
  uint64_t mark_src_uid = 0;       // ESDF: the source of the last fused update
  float mark_site_threshold = 0.0f;
  int xr_max_sq = 0, xr_cap_sq = 0;

  // Process-unique identity (never reused, unlike the address of a destroyed
  // layer).
  uint64_t uid = next_layer_uid();
  // ESDF: while every block came from mark_sites against the source layer
  // `subset_uid`, the block set is a subset of that TSDF layer's (so bounded
  // by its capacity).  Any call against another source, or any user write,
  // clears subset_valid for good (an empty layer starts over).
  uint64_t subset_uid = 0;
  bool subset_valid = true;
  // ESDF: user-written voxel data (vxm_layer_write_blocks) at any time, and the
  // largest max_sq any update used — together they decide whether every block
  // is in the lowering's compact sweep format (k_lower_xr FASTONLY)
  bool esdf_user_data = false;
  int esdf_max_sq_seen = 0;
  void note_esdf_source(const Layer* src) {
    if (num_blocks == 0) {
      subset_uid = src->uid;
      subset_valid = true;
    } else if (subset_uid != src->uid) {
      subset_valid = false;
    }
  }
  bool bounded_by(const Layer* src) const { return subset_valid && subset_uid == src->uid; }
  static uint64_t next_layer_uid();

  size_t voxel_bytes() const {
    return type == VXM_LAYER_ESDF ? 12 : type == VXM_LAYER_OCCUPANCY ? 4 : 8;  // TSDF, color: 8
  }
  size_t block_bytes() const { return voxel_bytes() * kVPB; }
  void* cur_pool() const { return pool[type == VXM_LAYER_ESDF ? cur_host : 0]; }
  // Grow pool/hash/side arrays so that capacity >= need (requires exact num_blocks).
  void ensure_capacity(uint64_t need);
  uint64_t limit() const { return max_blocks; }
  void refresh();  // sync + read meta (num_blocks, cur)
  // Enqueue a copy of the meta into the context status (read by sync_status)
  // and, after the sync, adopt it: one host round trip per API call.
  void stage_meta(int slot = 0);
  void adopt_meta(int slot = 0);
  ~Layer();
};

struct BlockList {
  Context* ctx = nullptr;
  DevBuf keys;                 // uint64 packed keys
  uint32_t* d_count = nullptr; // device count
  uint32_t cap = 0;            // capacity in keys (upper bound of count)
  uint32_t count_hint = 0;     // host upper bound of count
  std::vector<vxm_grid_index> host;
  bool host_valid = true;
  bool sorted_unique = false;  // keys are in strictly increasing GridIndex order
  // pinned host staging of assign_host (alive until the next assign, so the
  // upload is a true async DMA)
  uint64_t* staging = nullptr;
  uint64_t staging_cap = 0;
  // Host-bound results: the producer enqueues enqueue_host() before its one
  // status sync; a kernel unpacks the list into mapped pinned memory, so
  // fetch() needs no further round trip.
  bool want_host = false;
  bool host_pending = false;
  vxm_grid_index* mapped = nullptr;  // cudaHostAllocMapped, mapped_cap entries
  uint32_t* mapped_count = nullptr;
  uint32_t mapped_cap = 0;
  void enqueue_host();
  // Re-binds the list to context c; a context that still remembers this list
  // as its last host result forgets it (no dangling last_host_out).
  void bind(Context* c) {
    if (ctx && ctx != c && ctx->last_host_out == this) ctx->last_host_out = nullptr;
    ctx = c;
  }
  void ensure(uint32_t n);
  const std::vector<vxm_grid_index>& fetch();   // sync + download + unpack
  // upload (sorted as given); keep_host = false: no host copy kept (an input
  // list the caller never reads back)
  void assign_host(const vxm_grid_index* data, uint64_t n, bool keep_host = true);
  ~BlockList();
};

// Host-side loops over lists at least this long run on the host cores (OpenMP).
constexpr int64_t kHostParMin = 65536;

// The process-wide modification clock of the mark skip (Layer::stamp_mod).
uint32_t next_mod_tick();

struct EsdfState {
  std::vector<vxm_grid_index> lists[3];
};

// Launch with programmatic stream serialization (see pdl_wait in common.cuh);
// VXM_NO_PDL=1 falls back to plain launches.
bool pdl_enabled();
template <typename... P, typename... A>
inline void launch_pdl(cudaStream_t s, void (*k)(P...), dim3 g, dim3 b, size_t smem, A&&... args) {
  if (!pdl_enabled()) {
    k<<<g, b, smem, s>>>(std::forward<A>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  VXM_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...));
}

// ---- drivers (implemented in the kernel TUs) ----------------------------------
void diag_lidar_angles(Context* ctx, const double* xyz, uint64_t n, double* az, double* polar);  // integrate.cu
// view.cu — candidate blocks; when `alloc` != null the candidates are also
// looked up / allocated in that layer (fused allocation, integrator.cpp:84-87).
struct ViewArgs {
  vxm_pose T_LS;
  bool lidar;
  vxm_camera cam;
  vxm_lidar li;
  const float* depth_dev;
  int width, height;
  double block_size;
  vxm_view_config cfg;
};
// Returns the number of candidates only after ctx sync (status.n_candidates).
void run_view(Context* ctx, const ViewArgs& a, Layer* alloc, uint32_t* cand_cap_out);

// integrate.cu
void run_integrate(Layer* L, const ViewArgs& a, const vxm_integrator_config& cfg,
                   BlockList* changed_out);
// Split form for the fused frame update: launch (no sync) and, after the
// caller's sync, finish (checks + stats; false = pool grown, re-run the frame).
uint32_t integrate_launch(Layer* L, const ViewArgs& a, const vxm_integrator_config& cfg,
                          BlockList* changed_out);
bool integrate_finish(Layer* L, const ViewArgs& a, BlockList* changed_out, uint32_t nb_before);

// esdf.cu
void run_update_esdf(Layer* E, Layer* T, BlockList* updated, const vxm_esdf_config& cfg,
                     BlockList* changed_out);
void esdf_launch(Layer* E, Layer* T, BlockList* updated, const vxm_esdf_config& cfg,
                 BlockList* changed_out);
// shard.cu — one update_esdf over a block-sharded map (P shards, one context each)
void run_update_esdf_sharded(int P, Layer** E, Layer** T, BlockList** updated,
                             const vxm_esdf_config& cfg, int slab, BlockList** out);
void esdf_finish(Layer* E, BlockList* changed_out);
void run_mark_sites(Layer* E, Layer* T, BlockList* updated, const vxm_esdf_config& cfg,
                    EsdfState* st, std::vector<vxm_grid_index>* changed);
void run_clear_invalid(Layer* E, const vxm_esdf_config& cfg, EsdfState* st,
                       std::vector<vxm_grid_index>* changed);
int run_lower_esdf(Layer* E, EsdfState* st, const vxm_esdf_config& cfg,
                   std::vector<vxm_grid_index>* changed);
void esdf_sorted_export(Layer* E, std::vector<uint64_t>* keys, std::vector<int32_t>* slots);
// get_or_allocate of a sorted unique key list; slots in list order.
void alloc_key_list(Layer* L, BlockList* keys, int32_t* d_slots_out);

// query.cu
void run_query(Layer* E, const double* xyz_host, uint64_t n, int want_gradient, int interpolate,
               vxm_query_result* out_host);

// runtime.cu helpers used by the kernel TUs
void sort_unique_keys(Context* ctx, BlockList* list);  // device sort + unique (CUB)
void layer_export_sorted(Layer* L, std::vector<uint64_t>* keys, std::vector<int32_t>* slots);
void check_launch(Context* ctx, const char* what);
void host_trace_mark(const char* what);  // capi.cu (VXM_TRACE_HOST)
void host_trace_dev(Context* ctx, const char* what);

}  // namespace vxm
