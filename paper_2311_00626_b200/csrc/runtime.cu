// Host runtime: device memory management for layers (block pool + hash +
// ESDF side arrays), contexts, block lists and small device utilities.
#include <atomic>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "runtime.cuh"

namespace vxm {

// ---- DevBuf -------------------------------------------------------------------
void DevBuf::ensure(size_t n) {
  if (n <= bytes) return;
  release();
  size_t b = std::max<size_t>(n, 256);
  b = b + b / 4;  // slack so slowly growing sizes do not realloc every call
  VXM_CUDA(cudaMalloc(&p, b));
  bytes = b;
}
void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

void check_launch(Context* ctx, const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(VXM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  (void)ctx;
}

// ---- Context -------------------------------------------------------------------
uint64_t Layer::next_layer_uid() {
  static std::atomic<uint64_t> next{1};
  return next.fetch_add(1, std::memory_order_relaxed);
}

int Context::resident_per_sm(const void* kernel, int threads, size_t smem, int cap) {
  std::lock_guard<std::mutex> g(geo_mu);
  auto it = resident.find(kernel);
  if (it != resident.end()) return it->second;
  int bps = 0;
  VXM_CUDA(cudaSetDevice(device));
  VXM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, threads, smem));
  bps = std::max(1, std::min(bps, cap));
  resident.emplace(kernel, bps);
  return bps;
}

ScanTiles Context::next_scan(uint32_t tiles) {
  tiles = std::max<uint32_t>(tiles, 1);
  if (tiles > scan.cap) {
    // Grow both buffers (no pass is in flight across a host call boundary
    // once the stream is drained).
    VXM_CUDA(cudaStreamSynchronize(stream));
    for (int i = 0; i < 2; ++i) {
      if (scan.status[i]) cudaFree(scan.status[i]);
      VXM_CUDA(cudaMalloc(&scan.status[i], sizeof(unsigned long long) * tiles * 2));
      VXM_CUDA(cudaMemsetAsync(scan.status[i], 0, sizeof(unsigned long long) * tiles * 2, stream));
    }
    if (!scan.tickets) VXM_CUDA(cudaMalloc(&scan.tickets, sizeof(uint32_t) * 2));
    VXM_CUDA(cudaMemsetAsync(scan.tickets, 0, sizeof(uint32_t) * 2, stream));
    scan.cap = tiles * 2;
    scan.parity = 0;
  }
  ScanTiles st;
  const int p = scan.parity;
  st.status = scan.status[p];
  st.next = scan.status[1 - p];
  st.ticket = scan.tickets + p;
  st.next_ticket = scan.tickets + (1 - p);
  st.n_next = scan.cap;
  scan.parity = 1 - p;
  return st;
}

bool pdl_enabled() {
  static const bool on = std::getenv("VXM_NO_PDL") == nullptr;
  return on;
}

void Context::reset_status() {
  status_copies.clear();  // (copies queued by an operation that threw are dropped)
  if (!status_zero) VXM_CUDA(cudaMemsetAsync(d_status, 0, sizeof(DevStatus), stream));
  status_zero = false;  // the call's kernels write it from here on
}
struct WordCopies {
  const uint32_t* src[16];
  uint32_t* dst[16];
  int n;
};
__global__ void k_copy_words(WordCopies c) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < c.n) *c.dst[threadIdx.x] = *c.src[threadIdx.x];
}
void Context::flush_copies() {
  size_t i = 0;
  while (i < status_copies.size()) {
    WordCopies c{};
    for (; i < status_copies.size() && c.n < 16; ++i, ++c.n) {
      c.src[c.n] = status_copies[i].src;
      c.dst[c.n] = status_copies[i].dst;
    }
    launch_pdl(stream, k_copy_words, dim3(1), dim3(32), 0, c);
    count_launch();
  }
  status_copies.clear();
}
// The last queued word copies, then the whole status written straight into
// the mapped pinned host copy: the call's one host read needs no separate
// device-to-host DMA (whose small-copy latency is several microseconds).
constexpr int kStatusWords = int(sizeof(DevStatus) / sizeof(uint32_t));
static_assert(kStatusWords <= 32, "DevStatus fits one warp");
// k_emit_host's loop (the changed list unpacked into mapped pinned memory)
__device__ inline void emit_host(const Context::EmitHost& e) {
  const uint32_t n = min(*e.n_ptr, e.cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) *e.out_n = n;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t k = e.keys[i];
    e.out[i] = vxm_grid_index{key_x(k), key_y(k), key_z(k)};
  }
}
// CTA 0's first warp: the queued word copies, then the status into the host
// copy; every CTA: the deferred unpack of a host-bound list (if any)
__global__ void k_status_out(WordCopies c, uint32_t* __restrict__ st, uint32_t* __restrict__ host, int zero,
                             Context::EmitHost e) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    if (threadIdx.x < c.n) *c.dst[threadIdx.x] = *c.src[threadIdx.x];
    __syncwarp();
    if (threadIdx.x < kStatusWords) {
      host[threadIdx.x] = st[threadIdx.x];
      if (zero) st[threadIdx.x] = 0u;
    }
  }
  if (e.grid) emit_host(e);
}
void Context::sync_status(bool last) {
  // all but the last batch of queued copies, then the last batch + status out
  WordCopies tail{};
  size_t i = 0;
  while (status_copies.size() - i > 16) {
    WordCopies c{};
    for (; c.n < 16; ++i, ++c.n) {
      c.src[c.n] = status_copies[i].src;
      c.dst[c.n] = status_copies[i].dst;
    }
    launch_pdl(stream, k_copy_words, dim3(1), dim3(32), 0, c);
    count_launch();
  }
  for (; i < status_copies.size(); ++i, ++tail.n) {
    tail.src[tail.n] = status_copies[i].src;
    tail.dst[tail.n] = status_copies[i].dst;
  }
  status_copies.clear();
  const EmitHost e = emit;
  emit = EmitHost{};
  launch_pdl(stream, k_status_out, dim3(std::max<uint32_t>(e.grid, 1)), dim3(e.grid ? 256 : 32), 0, tail,
             reinterpret_cast<uint32_t*>(d_status), reinterpret_cast<uint32_t*>(h_status_dev), int(last), e);
  count_launch();
  VXM_CUDA(cudaStreamSynchronize(stream));
  status_zero = last;
  prof_resolve();
}

static cudaEvent_t take_event(Context* c) {
  if (!c->spare_events.empty()) {
    cudaEvent_t e = c->spare_events.back();
    c->spare_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  VXM_CUDA(cudaEventCreate(&e));
  return e;
}
void Context::prof_begin(const char* name) {
  if (!profile) return;
  prof_name = name;
  prof_a = take_event(this);
  VXM_CUDA(cudaEventRecord(prof_a, stream));
}
void Context::prof_end() {
  if (!profile || !prof_name) return;
  cudaEvent_t b = take_event(this);
  VXM_CUDA(cudaEventRecord(b, stream));
  pending.push_back({prof_name, prof_a, b});
  prof_name = nullptr;
}
void Context::prof_resolve() {
  for (const Pending& p : pending) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      auto& t = ktime[p.name];
      t.first += ms;
      t.second += 1;
    }
    spare_events.push_back(p.a);
    spare_events.push_back(p.b);
  }
  pending.clear();
}

// ---- Layer ---------------------------------------------------------------------
__global__ void k_rehash(HashView h, const uint64_t* slot_keys, uint32_t n) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x)
    hash_insert(h, slot_keys[s], int32_t(s));
}

template <typename T>
static void grow_copy(T** ptr, uint64_t old_elems, uint64_t live_elems, uint64_t new_elems,
                      int fill_byte, cudaStream_t st) {
  // Stream-ordered: the context's pool keeps freed memory (release
  // threshold = max), so growth costs the copy, not a cudaMalloc + device sync.
  T* np = nullptr;
  VXM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&np), sizeof(T) * std::max<uint64_t>(new_elems, 1), st));
  if (*ptr && live_elems)
    VXM_CUDA(cudaMemcpyAsync(np, *ptr, sizeof(T) * live_elems, cudaMemcpyDeviceToDevice, st));
  if (fill_byte >= 0 && new_elems > live_elems)
    VXM_CUDA(cudaMemsetAsync(np + live_elems, fill_byte, sizeof(T) * (new_elems - live_elems), st));
  if (*ptr) VXM_CUDA(cudaFreeAsync(*ptr, st));
  *ptr = np;
  (void)old_elems;
}

void Layer::refresh() {
  LayerMeta m;
  VXM_CUDA(cudaMemcpyAsync(&m, meta, sizeof m, cudaMemcpyDeviceToHost, ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  num_blocks = m.num_blocks;
  cur_host = m.cur;
}

void Layer::stage_meta(int slot) {
  ctx->queue_copy(&meta->num_blocks, slot ? &ctx->d_status->meta2_blocks : &ctx->d_status->meta_blocks, 2);
}
void Layer::adopt_meta(int slot) {
  num_blocks = slot ? ctx->h_status->meta2_blocks : ctx->h_status->meta_blocks;
  cur_host = slot ? ctx->h_status->meta2_cur : ctx->h_status->meta_cur;
}

void Layer::ensure_capacity(uint64_t need) {
  if (need <= capacity) return;
  static const bool trace = std::getenv("VXM_TRACE_GROW") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  const uint32_t cap_before = capacity;
  if (need > (uint64_t(1) << 31) - 1)
    throw Error(VXM_ERR_CAPACITY, "Layer: device block pool limit (2^31 blocks) exceeded");
  refresh();
  uint64_t nc = std::max<uint64_t>({need, uint64_t(capacity) * 2, 4096});
  nc = (nc + 1023) & ~uint64_t(1023);
  nc = std::min<uint64_t>(nc, std::max<uint64_t>(max_blocks, need));
  nc = std::max<uint64_t>(nc, need);
  cudaStream_t st = ctx->stream;
  if (num_blocks > capacity)
    throw Error(VXM_ERR_INTERNAL, "Layer: device block count exceeds the pool capacity");
  const uint64_t live = num_blocks;
  const size_t bb = block_bytes();
  // block pools (byte-typed); ESDF pool[1 - cur] is scratch for the next
  // full lowering, only its never-used tail must be zero.
  {
    unsigned char* p0 = static_cast<unsigned char*>(pool[0]);
    unsigned char* p1 = static_cast<unsigned char*>(pool[1]);
    const int c = type == VXM_LAYER_ESDF ? int(cur_host) : 0;
    unsigned char* pc = c ? p1 : p0;
    grow_copy(&pc, capacity * bb, live * bb, nc * bb, 0, st);
    if (type == VXM_LAYER_ESDF) {
      unsigned char* po = c ? p0 : p1;
      grow_copy(&po, capacity * bb, 0, nc * bb, 0, st);
      pool[c] = pc;
      pool[1 - c] = po;
    } else {
      pool[0] = pc;
    }
  }
  grow_copy(&slot_keys, capacity, live, nc, 0xFF, st);
  if (type == VXM_LAYER_TSDF || type == VXM_LAYER_OCCUPANCY) grow_copy(&stamp_mod, capacity, live, nc, 0, st);
  if (type == VXM_LAYER_ESDF) {
    grow_copy(&mark_stamp, capacity, live, nc, 0, st);
    grow_copy(&nbr, capacity * 6ull, live * 6ull, nc * 6ull, 0xFF, st);
    for (int i = 0; i < 2; ++i) {
      grow_copy(&sorted_keys[i], capacity, i == sorted_parity ? live : 0, nc, -1, st);
      grow_copy(&sorted_slots[i], capacity, i == sorted_parity ? live : 0, nc, -1, st);
      grow_copy(&stamp_dirty[i], capacity, live, nc, 0, st);
      grow_copy(&dirty_list[i], capacity, 0, nc, -1, st);
    }
    grow_copy(&stamp_mark, capacity, live, nc, 0, st);
    grow_copy(&stamp_new, capacity, live, nc, 0, st);
    grow_copy(&stamp_lchg, capacity, live, nc, 0, st);
    grow_copy(&line_mask, capacity * 3ull, live * 3ull, nc * 3ull, 0, st);
    grow_copy(&stamp_swept, capacity, live, nc, 0, st);
    grow_copy(&site_any, capacity, live, nc, 0, st);
    grow_copy(&site_near, capacity, 0, nc, -1, st);
    grow_copy(&r1_list, capacity * 3ull, 0, nc * 3ull, -1, st);
    for (int i = 0; i < 2; ++i) grow_copy(&dlist[i], capacity, 0, nc, 0, st);
    for (int i = 0; i < 3; ++i) grow_copy(&pair_face[i], capacity * 2ull, 0, nc * 2ull, 0, st);
    for (int a = 0; a < 3; ++a) grow_copy(&stamp_pair[a], capacity, live, nc, 0, st);
    grow_copy(&stamp_r1same, capacity, live, nc, 0, st);
    grow_copy(&stamp_quiet, capacity, live, nc, 0, st);
    ++esdf_gen;  // the scratch pool's blocks are not kept: no quiet block survives
  }
  // hash: power of two >= 2 * capacity, rebuilt from slot_keys
  uint64_t hc = 1024;
  while (hc < 2 * nc) hc <<= 1;
  if (hc != hash_cap) {
    if (hash.keys) VXM_CUDA(cudaFreeAsync(hash.keys, st));
    if (hash.vals) VXM_CUDA(cudaFreeAsync(hash.vals, st));
    VXM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&hash.keys), sizeof(uint64_t) * hc, st));
    VXM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&hash.vals), sizeof(int32_t) * hc, st));
    VXM_CUDA(cudaMemsetAsync(hash.keys, 0xFF, sizeof(uint64_t) * hc, st));
    hash.mask = uint32_t(hc - 1);
    hash_cap = uint32_t(hc);
    if (live) {
      k_rehash<<<std::min<uint32_t>(ceil_div(live, 256), 4096), 256, 0, st>>>(hash, slot_keys,
                                                                           uint32_t(live));
      ctx->count_launch();
      check_launch(ctx, "k_rehash");
    }
  }
  capacity = uint32_t(nc);
  if (trace) {
    VXM_CUDA(cudaStreamSynchronize(st));
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    std::fprintf(stderr, "[grow %s] %u -> %u blocks (need %llu, live %llu): %.2f ms\n",
                 type == VXM_LAYER_ESDF ? "esdf" : "tsdf", cap_before, capacity,
                 (unsigned long long)need, (unsigned long long)live, ms);
  }
}

Layer::~Layer() {
  for (void* p : {pool[0], pool[1]})
    if (p) cudaFree(p);
  if (hash.keys) cudaFree(hash.keys);
  if (hash.vals) cudaFree(hash.vals);
  if (slot_keys) cudaFree(slot_keys);
  if (meta) cudaFree(meta);
  if (nbr) cudaFree(nbr);
  for (int i = 0; i < 2; ++i) {
    if (sorted_keys[i]) cudaFree(sorted_keys[i]);
    if (sorted_slots[i]) cudaFree(sorted_slots[i]);
    if (stamp_dirty[i]) cudaFree(stamp_dirty[i]);
    if (dirty_list[i]) cudaFree(dirty_list[i]);
  }
  if (stamp_mark) cudaFree(stamp_mark);
  if (stamp_new) cudaFree(stamp_new);
  if (stamp_lchg) cudaFree(stamp_lchg);
  if (dirty_count) cudaFree(dirty_count);
  if (line_mask) cudaFree(line_mask);
  if (stamp_swept) cudaFree(stamp_swept);
  if (site_any) cudaFree(site_any);
  if (site_near) cudaFree(site_near);
  if (r1_list) cudaFree(r1_list);
  for (unsigned long long* p : dlist)
    if (p) cudaFree(p);
  for (unsigned long long* p : pair_face)
    if (p) cudaFree(p);
  for (uint32_t* p : stamp_pair)
    if (p) cudaFree(p);
  if (stamp_r1same) cudaFree(stamp_r1same);
  if (stamp_quiet) cudaFree(stamp_quiet);
  if (stamp_mod) cudaFree(stamp_mod);
  if (mark_stamp) cudaFree(mark_stamp);
}

uint32_t next_mod_tick() {
  static std::atomic<uint32_t> clock{0};
  return clock.fetch_add(1u, std::memory_order_relaxed) + 1u;
}

// ---- BlockList -----------------------------------------------------------------
void BlockList::ensure(uint32_t n) {
  if (ctx && ctx->emit.list == this) ctx->flush_emit();  // (its keys may move)
  if (!d_count) {
    VXM_CUDA(cudaMalloc(&d_count, sizeof(uint32_t)));
    VXM_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), ctx->stream));
  }
  if (n > cap) {
    // preserve nothing: lists are rewritten by their producer
    keys.ensure(sizeof(uint64_t) * std::max<uint32_t>(n, 1));
    cap = uint32_t(keys.bytes / sizeof(uint64_t));
  }
}

__global__ void k_emit_host(Context::EmitHost e) {
  pdl_wait();
  pdl_trigger();
  emit_host(e);
}

void Context::flush_emit() {
  if (!emit.grid) return;
  const EmitHost e = emit;
  emit = EmitHost{};
  launch_pdl(stream, k_emit_host, dim3(e.grid), dim3(256), 0, e);
  count_launch();
  check_launch(this, "k_emit_host");
}

void BlockList::enqueue_host() {
  ctx->flush_emit();  // one deferred unpack at a time (and before mapped may move)
  const uint32_t need = std::max<uint32_t>(count_hint, 1);
  if (need > mapped_cap) {
    if (mapped) VXM_CUDA(cudaFreeHost(mapped));
    mapped_cap = std::max<uint32_t>(need, 4096);
    VXM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&mapped), sizeof(vxm_grid_index) * mapped_cap,
                           cudaHostAllocMapped));
  }
  if (!mapped_count)
    VXM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&mapped_count), sizeof(uint32_t), cudaHostAllocMapped));
  const uint32_t grid = std::min<uint32_t>(ceil_div(need, 256), uint32_t(ctx->sm_count));
  ctx->emit = Context::EmitHost{keys.as<const uint64_t>(), static_cast<const uint32_t*>(d_count), mapped,
                                mapped_count, mapped_cap, std::max<uint32_t>(grid, 1), this};
  host_pending = true;
}

// dst = src[0, n): large lists copied by the host cores in parallel
static void host_copy(std::vector<vxm_grid_index>& dst, const vxm_grid_index* src, uint64_t n) {
  dst.resize(n);
  const int64_t nn = int64_t(n);
  if (nn < kHostParMin) {
    if (n) std::memcpy(dst.data(), src, sizeof(vxm_grid_index) * n);
    return;
  }
  constexpr int64_t kChunk = 16384;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nn; c += kChunk)
    std::memcpy(dst.data() + c, src + c, sizeof(vxm_grid_index) * size_t(std::min(kChunk, nn - c)));
}

const std::vector<vxm_grid_index>& BlockList::fetch() {
  if (host_valid) return host;
  if (host_pending) {  // unpacked by k_emit_host / k_status_out into mapped memory
    if (ctx->emit.list == this) ctx->flush_emit();
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint32_t n = *mapped_count;
    host_copy(host, mapped, n);
    host_pending = false;
    host_valid = true;
    count_hint = n;
    return host;
  }
  uint32_t n = 0;
  if (d_count) {
    VXM_CUDA(cudaMemcpyAsync(&n, d_count, sizeof n, cudaMemcpyDeviceToHost, ctx->stream));
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  std::vector<uint64_t> k(n);
  if (n) {
    VXM_CUDA(cudaMemcpyAsync(k.data(), keys.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost,
                             ctx->stream));
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  host.resize(n);
  for (uint32_t i = 0; i < n; ++i) host[i] = {key_x(k[i]), key_y(k[i]), key_z(k[i])};
  host_valid = true;
  count_hint = n;
  return host;
}

void BlockList::assign_host(const vxm_grid_index* data, uint64_t n, bool keep_host) {
  ensure(uint32_t(std::max<uint64_t>(n, 1)));
  host_pending = false;
  if (n + 1 > staging_cap) {
    if (staging) {
      VXM_CUDA(cudaStreamSynchronize(ctx->stream));  // a previous upload may still read it
      VXM_CUDA(cudaFreeHost(staging));
    }
    staging_cap = std::max<uint64_t>(n + 1, 4096);
    VXM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&staging), sizeof(uint64_t) * staging_cap));
  }
  // range check + packing, then the order check (input validation only):
  // branch-free, and over the host cores for large lists (C5: 262k keys)
  const int64_t nn = int64_t(n);
  uint32_t bad = 0, unsorted = 0;
#pragma omp parallel for schedule(static) reduction(| : bad) if (nn >= kHostParMin)
  for (int64_t i = 0; i < nn; ++i) {
    const vxm_grid_index g = data[i];
    bad |= uint32_t(!coord_ok(g.x)) | uint32_t(!coord_ok(g.y)) | uint32_t(!coord_ok(g.z));
    staging[i] = pack_key(g.x, g.y, g.z);
  }
  if (bad) throw Error(VXM_ERR_INVALID_ARGUMENT, "block index outside the supported range (+-2^20)");
#pragma omp parallel for schedule(static) reduction(| : unsorted) if (nn >= kHostParMin)
  for (int64_t i = 1; i < nn; ++i) unsorted |= uint32_t(staging[i - 1] >= staging[i]);
  const bool sorted = unsorted == 0u;
  staging[n] = n;  // count travels in the same copy (low 32 bits)
  const uint32_t n32 = uint32_t(n);
  VXM_CUDA(cudaMemcpyAsync(keys.p, staging, sizeof(uint64_t) * n, cudaMemcpyHostToDevice,
                           ctx->stream));
  VXM_CUDA(cudaMemcpyAsync(d_count, &staging[n], sizeof(uint32_t), cudaMemcpyHostToDevice,
                           ctx->stream));
  // staging (pinned) stays alive until the next assign; calls that reuse the
  // list synchronise the stream before returning
  if (keep_host) {
    host_copy(host, data, n);
    host_valid = true;
  } else {
    host.clear();
    host_valid = false;  // (fetch() downloads it if ever asked)
  }
  count_hint = n32;
  sorted_unique = sorted;
}

BlockList::~BlockList() {
  if (ctx && ctx->last_host_out == this) ctx->last_host_out = nullptr;
  if (ctx && ctx->emit.list == this) ctx->emit = Context::EmitHost{};  // (nobody reads it)
  if (ctx && (staging || mapped)) cudaStreamSynchronize(ctx->stream);
  if (staging) cudaFreeHost(staging);
  if (mapped) cudaFreeHost(mapped);
  if (mapped_count) cudaFreeHost(mapped_count);
  keys.release();
  if (d_count) cudaFree(d_count);
}

// ---- sorting utilities (API paths only; the hot path never sorts) ---------------
__global__ void k_count_to_dev(uint32_t* dst, const int* src) { *dst = uint32_t(*src); }

void sort_unique_keys(Context* ctx, BlockList* list) {
  const uint32_t n = list->count_hint;
  if (n <= 1) return;
  DevBuf& t0 = ctx->tmp[0];
  t0.ensure(sizeof(uint64_t) * n);
  size_t sort_bytes = 0, uniq_bytes = 0;
  uint64_t* keys = list->keys.as<uint64_t>();
  cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, keys, t0.as<uint64_t>(), int(n), 0, 63,
                                 ctx->stream);
  cub::DeviceSelect::Unique(nullptr, uniq_bytes, t0.as<uint64_t>(), keys, (int*)nullptr, int(n),
                            ctx->stream);
  const size_t work = (std::max(sort_bytes, uniq_bytes) + 255) & ~size_t(255);
  ctx->cub_tmp.ensure(work + 256);
  int* d_nsel = reinterpret_cast<int*>(static_cast<char*>(ctx->cub_tmp.p) + work);
  VXM_CUDA(cub::DeviceRadixSort::SortKeys(ctx->cub_tmp.p, sort_bytes, keys, t0.as<uint64_t>(),
                                          int(n), 0, 63, ctx->stream));
  VXM_CUDA(cub::DeviceSelect::Unique(ctx->cub_tmp.p, uniq_bytes, t0.as<uint64_t>(), keys, d_nsel,
                                     int(n), ctx->stream));
  k_count_to_dev<<<1, 1, 0, ctx->stream>>>(list->d_count, d_nsel);
  ctx->count_launch(3);
  check_launch(ctx, "sort_unique_keys");
  list->host_valid = false;
  list->host_pending = false;
}

// Sorted (key, slot) export of a TSDF layer (sorted_indices, layer.hpp:109-117).
__global__ void k_iota_keys(const uint64_t* slot_keys, uint64_t* keys, int32_t* slots, uint32_t n) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    keys[s] = slot_keys[s];
    slots[s] = int32_t(s);
  }
}

void layer_export_sorted(Layer* L, std::vector<uint64_t>* keys, std::vector<int32_t>* slots) {
  Context* ctx = L->ctx;
  L->refresh();
  const uint32_t n = L->num_blocks;
  keys->resize(n);
  slots->resize(n);
  if (!n) return;
  if (L->type == VXM_LAYER_ESDF) {
    esdf_sorted_export(L, keys, slots);
    return;
  }
  for (int i = 0; i < 4; ++i) ctx->tmp[i].ensure(sizeof(uint64_t) * n);
  uint64_t* k_in = ctx->tmp[0].as<uint64_t>();
  uint64_t* k_out = ctx->tmp[1].as<uint64_t>();
  int32_t* v_in = ctx->tmp[2].as<int32_t>();
  int32_t* v_out = ctx->tmp[3].as<int32_t>();
  k_iota_keys<<<std::min<uint32_t>(ceil_div(n, 256), 4096), 256, 0, ctx->stream>>>(L->slot_keys,
                                                                                  k_in, v_in, n);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k_in, k_out, v_in, v_out, int(n), 0, 63,
                                  ctx->stream);
  ctx->cub_tmp.ensure(bytes);
  VXM_CUDA(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, bytes, k_in, k_out, v_in, v_out, int(n),
                                           0, 63, ctx->stream));
  ctx->count_launch(2);
  check_launch(ctx, "layer_export_sorted");
  VXM_CUDA(cudaMemcpyAsync(keys->data(), k_out, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost,
                           ctx->stream));
  VXM_CUDA(cudaMemcpyAsync(slots->data(), v_out, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                           ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace vxm
