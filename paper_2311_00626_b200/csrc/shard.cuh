// Sharded ESDF update: per-shard state and steps (shard.cu), shared with the
// step C-ABI (capi.cu).
#pragma once

#include "esdf_host.cuh"

namespace vxm {

// Exchange buffer of n boundary blocks (one contiguous allocation, so one
// transfer per neighbour): keys [8n] | dirty bytes [n, padded to 8] | faces
// [n][2][64][3] words.
inline size_t pad8(size_t n) { return (n + 7) & ~size_t(7); }
inline size_t xbuf_bytes(uint32_t n) { return 8ull * n + pad8(n) + 1536ull * n; }
struct XView {
  uint64_t* keys;
  uint8_t* dirty;
  uint32_t* faces;
};
inline XView xview(void* base, uint32_t n) {
  unsigned char* b = static_cast<unsigned char*>(base);
  return XView{reinterpret_cast<uint64_t*>(b), b + 8ull * n,
               reinterpret_cast<uint32_t*>(b + 8ull * n + pad8(n))};
}

struct ShardUpdate {
  Layer* E = nullptr;
  Layer* T = nullptr;
  Context* ctx = nullptr;
  int rank = 0, world = 1, slab = 1;
  BlockList uni;  // union of the shards' updated lists (sorted, unique)
  EsdfScratch s{};
  uint32_t epoch = 0, n_all_cap = 0, base = 0, cur = 0, n_blocks = 0;
  uint32_t n_bnd = 0, n_rcv[2] = {0, 0}, n_dirty = 0, rounds = 0;
  bool local_any = false;
  DevBuf ctr, bnd_keys, bnd_slots, bnd_flags, bnd_n, cub_tmp, snd, rcv[2];
  LowerArgs la{};
  LayerMeta* h_meta = nullptr;  // pinned: the layer meta after the mark phase
  uint32_t* h_cnt = nullptr;    // pinned: [0] boundary blocks, [1] next dirty count
  cudaEvent_t ev = nullptr;     // in-process exchange ordering
  DevBuf mbox;                  // fused exchange: receive flags, count board, go, rounds
  bool fused = false;           // the round loop ran in k_shard_fused (rounds on the device)
  std::vector<void*> ipc_open;  // peer allocations opened for the fused multi-process exchange
  ShardUpdate() = default;
  ShardUpdate(const ShardUpdate&) = delete;
  ShardUpdate& operator=(const ShardUpdate&) = delete;
  ~ShardUpdate();
};

// Steps: *_launch enqueue on the shard's context stream; the plain forms also
// synchronise (the step C-ABI).
void shard_begin(ShardUpdate& x, const vxm_esdf_config& cfg);
void shard_plan(ShardUpdate& x);
void shard_set_neighbours(ShardUpdate& x, uint32_t n_left, uint32_t n_right);
void shard_sweep(ShardUpdate& x, uint32_t r);  // enqueue only
void shard_border_launch(ShardUpdate& x, uint32_t r);
uint32_t shard_border(ShardUpdate& x, uint32_t r);
uint32_t* next_count_ptr(ShardUpdate& x, uint32_t r);
void shard_finish(ShardUpdate& x, bool lowered, BlockList* out);
// Fused multi-process exchange over CUDA IPC: this rank's handles (rcv[0],
// rcv[1], mailbox; 3 x 64 bytes — also clears the mailbox, so call before the
// all-gather that acts as the barrier) and the launch of the round loop.
void shard_ipc_handles(ShardUpdate& x, void* out192);
void shard_lower_fused_ipc(ShardUpdate& x, const void* all_handles, int ranks_on_device);

}  // namespace vxm
