// extern "C" boundary of libvoxmap_b200 (include/voxmap_b200.h).
//
// Each entry point validates its arguments exactly where the reference does
// (before any mutation), maps C++ errors onto vxm_status codes that mirror
// the reference's exception types, and dispatches to the device drivers.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <tuple>
#include <string>
#include <vector>

#include "runtime.cuh"
#include "mesh.cuh"
#include "shard.cuh"

using namespace vxm;

struct vxm_context : Context {};
struct vxm_layer : Layer {};
struct vxm_blocklist : BlockList {};
struct vxm_esdf_state : EsdfState {};
struct vxm_mesh_layer : MeshLayerH {};

namespace {
thread_local std::string g_err;

template <typename F>
vxm_status guard(F&& f) {
  try {
    f();
    return VXM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return vxm_status(e.code);
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return VXM_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VXM_ERR_INTERNAL;
  }
}

#define REQUIRE_ARG(cond, msg) \
  do {                         \
    if (!(cond)) throw Error(VXM_ERR_INVALID_ARGUMENT, msg); \
  } while (0)

inline double sum3h(double a0, double a1, double a2) { return a0 + (a1 + a2); }

__global__ void k_gather_blocks(const unsigned char* pool, const int32_t* slots, uint32_t n,
                                uint32_t block_bytes, unsigned char* out) {
  const uint32_t words = block_bytes / 4;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < uint64_t(n) * words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t b = uint32_t(i / words), w = uint32_t(i % words);
    const int32_t s = slots[b];
    reinterpret_cast<uint32_t*>(out)[i] =
        s >= 0 ? reinterpret_cast<const uint32_t*>(pool + size_t(s) * block_bytes)[w] : 0u;
  }
}
__global__ void k_scatter_blocks(unsigned char* pool, const int32_t* slots, uint32_t n,
                                 uint32_t block_bytes, const unsigned char* in) {
  const uint32_t words = block_bytes / 4;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < uint64_t(n) * words;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t b = uint32_t(i / words), w = uint32_t(i % words);
    const int32_t s = slots[b];
    if (s >= 0)
      reinterpret_cast<uint32_t*>(pool + size_t(s) * block_bytes)[w] =
          reinterpret_cast<const uint32_t*>(in)[i];
  }
}
__global__ void k_mark_site_any(uint8_t* site_any, const int32_t* slots, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (slots[i] >= 0) site_any[slots[i]] = 1;  // user data: may hold sites
}
__global__ void k_lookup(const uint64_t* keys, uint32_t n, HashView h, int32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = h.keys ? hash_find(h, keys[i]) : -1;
}

uint32_t grid1d(Context* ctx, uint64_t n) {
  return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(ctx->sm_count) * 8)));
}

void lookup_host_keys(Layer* L, const vxm_grid_index* keys, uint64_t n, std::vector<int32_t>* slots,
                      DevBuf* dslots) {
  Context* ctx = L->ctx;
  std::vector<uint64_t> k(n);
  for (uint64_t i = 0; i < n; ++i) {
    const bool ok = coord_ok(keys[i].x) && coord_ok(keys[i].y) && coord_ok(keys[i].z);
    k[i] = ok ? pack_key(keys[i].x, keys[i].y, keys[i].z) : kEmptyKey - 1;  // never present
  }
  DevBuf dk;
  dk.ensure(sizeof(uint64_t) * std::max<uint64_t>(n, 1));
  dslots->ensure(sizeof(int32_t) * std::max<uint64_t>(n, 1));
  if (n) {
    VXM_CUDA(cudaMemcpyAsync(dk.p, k.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice, ctx->stream));
    k_lookup<<<grid1d(ctx, n), 256, 0, ctx->stream>>>(dk.as<uint64_t>(), uint32_t(n), L->hash,
                                                     dslots->as<int32_t>());
    ctx->count_launch();
    check_launch(ctx, "k_lookup");
  }
  slots->resize(n);
  if (n)
    VXM_CUDA(cudaMemcpyAsync(slots->data(), dslots->p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                             ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void ensure_sorted_unique(vxm_blocklist* list) {
  if (list->sorted_unique) return;
  sort_unique_keys(list->ctx, list);
  // count after unique is on the device; count_hint stays an upper bound
  list->sorted_unique = true;
}

// The ESDF's source layer: Layer<TsdfVoxel> or Layer<OccupancyVoxel>
// (esdf/integrator.hpp:81-120 overloads).
bool is_source(const vxm_layer* L) {
  return L->type == VXM_LAYER_TSDF || L->type == VXM_LAYER_OCCUPANCY;
}

// VXM_TRACE_HOST=1: host-side phase times of the host-buffer entry points (µs).
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0;
  char buf[256];
  int len = 0;
  explicit HostTrace(const char* name) : on(std::getenv("VXM_TRACE_HOST") != nullptr) {
    if (on) {
      t0 = std::chrono::steady_clock::now();
      len = std::snprintf(buf, sizeof buf, "%s:", name);
      g_host_trace = this;
    }
  }
  // device-side marks (events on the context stream), printed at the end
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8];
  const char* ev_name[8];
  int n_ev = 0;
  void dev_mark(cudaStream_t s, const char* what) {
    if (!on || n_ev >= 8) return;
    stream = s;
    cudaEventCreate(&ev[n_ev]);
    cudaEventRecord(ev[n_ev], s);
    ev_name[n_ev++] = what;
  }
  void mark(const char* what) {
    if (!on || len >= int(sizeof buf) - 32) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    len += std::snprintf(buf + len, sizeof buf - len, " %s %.1f", what, us);
  }
  ~HostTrace() {
    if (on) {
      if (n_ev > 1) {
        cudaStreamSynchronize(stream);
        len += std::snprintf(buf + len, sizeof buf - len, " | dev");
        for (int i = 1; i < n_ev && len < int(sizeof buf) - 32; ++i) {
          float ms = 0.0f;
          cudaEventElapsedTime(&ms, ev[0], ev[i]);
          len += std::snprintf(buf + len, sizeof buf - len, " %s %.1f", ev_name[i], 1e3 * ms);
        }
      }
      for (int i = 0; i < n_ev; ++i) cudaEventDestroy(ev[i]);
      std::fprintf(stderr, "%s\n", buf);
      g_host_trace = nullptr;
    }
  }
  static thread_local HostTrace* g_host_trace;
};
thread_local HostTrace* HostTrace::g_host_trace = nullptr;

void check_pose(const vxm_pose* T) {
  if (!vxm_pose_valid(T)) throw Error(VXM_ERR_INVALID_POSE, "integrate: degenerate sensor pose");
}

void stage_depth(Context* ctx, const float* depth, int w, int h, bool on_device, const float** out) {
  const size_t bytes = sizeof(float) * size_t(w) * size_t(h);
  if (on_device) {
    *out = depth;
    return;
  }
  ctx->depth.ensure(std::max<size_t>(bytes, 4));
  if (bytes)
    VXM_CUDA(cudaMemcpyAsync(ctx->depth.p, depth, bytes, cudaMemcpyHostToDevice, ctx->stream));
  *out = ctx->depth.as<float>();
}

// check_frame — integrator.cpp:26-34 (before any mutation) + view arguments.
ViewArgs frame_args(vxm_layer* L, const float* depth, int w, int h, const vxm_pose* T,
                    const vxm_camera* cam, const vxm_lidar* li, const vxm_integrator_config* cfg,
                    bool on_device) {
  REQUIRE_ARG(L->type == VXM_LAYER_TSDF || L->type == VXM_LAYER_OCCUPANCY,
              "integrate: layer is not a TSDF or occupancy layer");
  check_pose(T);
  const int sw = cam ? cam->width : li->num_azimuth;
  const int sh = cam ? cam->height : li->num_elevation;
  if (w != sw || h != sh)
    throw Error(VXM_ERR_INVALID_ARGUMENT, "integrate: image size does not match intrinsics");
  REQUIRE_ARG(w == 0 || h == 0 || depth, "integrate: null depth image");
  ViewArgs va{};
  va.T_LS = *T;
  va.lidar = li != nullptr;
  if (cam) va.cam = *cam;
  if (li) va.li = *li;
  va.width = w;
  va.height = h;
  va.block_size = L->vs * kVPS;
  va.cfg = {cfg->max_integration_distance, cfg->truncation, cfg->view_pixel_subsample};
  stage_depth(L->ctx, depth, w, h, on_device, &va.depth_dev);
  return va;
}

vxm_status integrate_common(vxm_layer* L, const float* depth, int w, int h, const vxm_pose* T,
                            const vxm_camera* cam, const vxm_lidar* li,
                            const vxm_integrator_config* cfg, vxm_blocklist* out, bool on_device) {
  return guard([&] {
    REQUIRE_ARG(L && T && cfg && out && (cam || li), "integrate: null argument");
    HostTrace tr("integrate");
    tr.dev_mark(L->ctx->stream, "start");
    const ViewArgs va = frame_args(L, depth, w, h, T, cam, li, cfg, on_device);
    tr.mark("staged");
    tr.dev_mark(L->ctx->stream, "h2d");
    out->bind(L->ctx);
    out->want_host = !on_device;  // unpacked to mapped host memory before the one sync
    try {
      run_integrate(L, va, *cfg, out);
    } catch (...) {
      out->want_host = false;
      throw;
    }
    tr.mark("synced");
    out->want_host = false;
    out->sorted_unique = true;
    if (!on_device) {
      out->fetch();
      L->ctx->last_host_out = out;
    }
    tr.mark("fetched");
  });
}

// One frame of the replay pipeline (pipeline.cpp:95-108): integrate_depth,
// then update_esdf on its changed list, enqueued back to back with a single
// host round trip for both (status, errors, metas).  A TSDF pool overflow
// touches no voxel and leaves the ESDF update empty, so the frame is re-run
// after the pool grows.
vxm_status frame_common(vxm_layer* T, vxm_layer* E, const float* depth, int w, int h,
                        const vxm_pose* pose, const vxm_camera* cam, const vxm_lidar* li,
                        const vxm_integrator_config* icfg, const vxm_esdf_config* ecfg,
                        vxm_blocklist* tout, vxm_blocklist* eout) {
  return guard([&] {
    REQUIRE_ARG(T && pose && icfg && tout && (cam || li), "update_frame: null argument");
    if (E) {
      REQUIRE_ARG(ecfg && eout, "update_frame: null ESDF argument");
      REQUIRE_ARG(E->type == VXM_LAYER_ESDF, "update_esdf: expects (ESDF layer, TSDF or occupancy layer)");
      REQUIRE_ARG(E->ctx == T->ctx, "update_frame: layers on different contexts");
      if (E->vs != T->vs)
        throw Error(VXM_ERR_INVALID_ARGUMENT, "update_esdf: source and ESDF layer voxel sizes differ");
    }
    const ViewArgs va = frame_args(T, depth, w, h, pose, cam, li, icfg, true);
    Context* ctx = T->ctx;
    tout->bind(ctx);
    if (E) eout->bind(ctx);
    for (int attempt = 0; attempt < 4; ++attempt) {
      ctx->reset_status();
      const uint32_t nb_before = T->num_blocks;
      integrate_launch(T, va, *icfg, tout);
      tout->sorted_unique = true;
      if (E) esdf_launch(E, T, tout, *ecfg, eout);
      T->stage_meta(0);
      if (E) E->stage_meta(1);
      ctx->sync_status(true);
      T->adopt_meta(0);
      if (E) E->adopt_meta(1);
      if (!integrate_finish(T, va, tout, nb_before)) continue;
      if (E) {
        esdf_finish(E, eout);
        eout->sorted_unique = true;
      }
      return;
    }
    throw Error(VXM_ERR_INTERNAL, "update_frame: pool growth did not converge");
  });
}

}  // namespace

namespace vxm {
void host_trace_mark(const char* what) {
  if (HostTrace::g_host_trace) HostTrace::g_host_trace->mark(what);
}
void host_trace_dev(Context* ctx, const char* what) {
  if (HostTrace::g_host_trace) HostTrace::g_host_trace->dev_mark(ctx->stream, what);
}
}  // namespace vxm

extern "C" {

const char* vxm_last_error(void) { return g_err.c_str(); }
const char* vxm_version(void) { return "voxmap_b200 0.1 (sm_100a)"; }

void vxm_integrator_config_default(vxm_integrator_config* c) {
  auto q = [](float v) { return float(std::nearbyint(double(v) * 4096.0) / 4096.0); };
  c->truncation = 0.2;
  c->max_weight = 100.0f;
  c->weighting = VXM_WEIGHT_CONSTANT;
  c->max_integration_distance = 5.0;
  c->camera_sample = VXM_SAMPLE_NEAREST;
  c->lidar_sample = VXM_SAMPLE_LINEAR;
  c->max_sample_gap = 0.2f;
  c->view_pixel_subsample = 8;
  c->hit_log_odds = q(0.8473f);
  c->miss_log_odds = q(-0.4055f);
  c->log_odds_min = -5.0f;
  c->log_odds_max = 5.0f;
  c->parallel = 1;
}
void vxm_esdf_config_default(vxm_esdf_config* c) {
  c->site_threshold = 0.05;
  c->occupied_log_odds_threshold = 0.0f;
  c->max_distance = 2.0;
  c->parallel = 1;
}
void vxm_query_config_default(vxm_query_config* c) {
  c->interpolate = 1;
  c->parallel = 1;
}

// Pose::valid — pose.hpp:42-50 (same association order as the oracle shim).
int vxm_pose_valid(const vxm_pose* T) {
  for (int i = 0; i < 9; ++i)
    if (!std::isfinite(T->R[i])) return 0;
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(T->t[i])) return 0;
  const double* m = T->R;
  auto M = [m](int r, int c) { return m[r * 3 + c]; };
  const double h012 = M(0, 0) * (M(1, 1) * M(2, 2) - M(1, 2) * M(2, 1));
  const double h102 = M(0, 1) * (M(1, 0) * M(2, 2) - M(1, 2) * M(2, 0));
  const double h201 = M(0, 2) * (M(1, 0) * M(2, 1) - M(1, 1) * M(2, 0));
  const double det = h012 - h102 + h201;
  double ortho = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      const double v = sum3h(M(0, r) * M(0, c), M(1, r) * M(1, c), M(2, r) * M(2, c)) -
                       (r == c ? 1.0 : 0.0);
      ortho = std::max(ortho, std::fabs(v));
    }
  return std::fabs(det - 1.0) <= 1e-6 && ortho <= 1e-6;
}
// Pose::inverse — pose.hpp:52
void vxm_pose_inverse(const vxm_pose* T, vxm_pose* out) {
  vxm_pose o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.R[3 * r + c] = T->R[3 * c + r];
  for (int i = 0; i < 3; ++i)
    o.t[i] = -sum3h(o.R[3 * i] * T->t[0], o.R[3 * i + 1] * T->t[1], o.R[3 * i + 2] * T->t[2]);
  *out = o;
}

vxm_status vxm_context_create(int device, vxm_context** out) {
  return guard([&] {
    REQUIRE_ARG(out, "null out");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0)
      throw Error(VXM_ERR_CUDA, "voxmap_b200: no CUDA device " + std::to_string(device) +
                                    " (this library has no CPU fallback)");
    cudaDeviceProp prop{};
    VXM_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw Error(VXM_ERR_CUDA, std::string("voxmap_b200 requires an sm_100 (B200) device, got ") +
                                    prop.name);
    VXM_CUDA(cudaSetDevice(device));
    auto* ctx = new vxm_context();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    VXM_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    {  // layer pools grow stream-ordered from the device pool; keep what is freed
      cudaMemPool_t mp;
      VXM_CUDA(cudaDeviceGetDefaultMemPool(&mp, device));
      uint64_t keep = ~uint64_t(0);
      VXM_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    VXM_CUDA(cudaMalloc(&ctx->d_status, sizeof(DevStatus)));
    VXM_CUDA(cudaHostAlloc(&ctx->h_status, sizeof(DevStatus), cudaHostAllocMapped));
    VXM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->h_status_dev), ctx->h_status, 0));
    // The context stream is non-blocking: every initialisation is ordered on
    // it, never on the legacy stream (which it does not synchronise with).
    VXM_CUDA(cudaMemsetAsync(ctx->d_status, 0, sizeof(DevStatus), ctx->stream));
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = ctx;
  });
}

void vxm_context_destroy(vxm_context* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  for (int i = 0; i < 2; ++i)
    if (ctx->scan.status[i]) cudaFree(ctx->scan.status[i]);
  if (ctx->scan.tickets) cudaFree(ctx->scan.tickets);
  delete static_cast<vxm_blocklist*>(ctx->scratch_in);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

vxm_status vxm_context_synchronize(vxm_context* ctx) {
  return guard([&] {
    ctx->sync_status();
    const DevStatus& s = *ctx->h_status;
    if (s.bitmap_overflow) throw Error(VXM_ERR_INTERNAL, "candidate bitmap overflow");
    if (s.capacity_error || s.pool_overflow)
      throw Error(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
  });
}

vxm_status vxm_context_set_shard(vxm_context* ctx, int rank, int world, int slab) {
  return guard([&] {
    REQUIRE_ARG(world >= 1 && rank >= 0 && rank < world && slab >= 1, "invalid shard");
    ctx->rank = rank;
    ctx->world = world;
    ctx->slab = slab;
  });
}
uint64_t vxm_context_launch_count(const vxm_context* ctx) { return ctx ? ctx->launches : 0; }
uint64_t vxm_context_stream(const vxm_context* ctx) {
  return ctx ? reinterpret_cast<uint64_t>(ctx->stream) : 0;
}
vxm_status vxm_context_stats(vxm_context* ctx, vxm_stats* out) {
  return guard([&] { *out = ctx->stats; });
}
void vxm_context_reset_stats(vxm_context* ctx) {
  if (ctx) ctx->stats = vxm_stats{};
}
vxm_status vxm_context_set_profiling(vxm_context* ctx, int enable) {
  return guard([&] {
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->prof_resolve();
    ctx->profile = enable != 0;
  });
}
vxm_status vxm_context_kernel_time(vxm_context* ctx, const char* kernel, double* ms,
                                   uint64_t* launches) {
  return guard([&] {
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->prof_resolve();
    auto it = ctx->ktime.find(kernel ? kernel : "");
    *ms = it == ctx->ktime.end() ? 0.0 : it->second.first;
    *launches = it == ctx->ktime.end() ? 0 : it->second.second;
  });
}
vxm_status vxm_diag_lidar_angles(vxm_context* ctx, const double* xyz, uint64_t n, double* azimuth,
                                 double* polar) {
  return guard([&] {
    REQUIRE_ARG(ctx && (n == 0 || (xyz && azimuth && polar)), "diag_lidar_angles: null argument");
    diag_lidar_angles(ctx, xyz, n, azimuth, polar);
  });
}
void vxm_context_reset_kernel_times(vxm_context* ctx) {
  if (ctx) ctx->ktime.clear();
}

vxm_status vxm_host_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    REQUIRE_ARG(out, "null argument");
    *out = nullptr;
    VXM_CUDA(cudaHostAlloc(out, std::max<uint64_t>(bytes, 1), cudaHostAllocDefault));
  });
}
void vxm_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

vxm_status vxm_blocklist_create(vxm_context* ctx, vxm_blocklist** out) {
  return guard([&] {
    auto* l = new vxm_blocklist();
    l->ctx = ctx;
    l->ensure(1);
    *out = l;
  });
}
void vxm_blocklist_destroy(vxm_blocklist* l) { delete l; }
vxm_status vxm_blocklist_host(vxm_blocklist* l, const vxm_grid_index** data, uint64_t* n) {
  return guard([&] {
    const auto& h = l->fetch();
    *data = h.data();
    *n = h.size();
  });
}
vxm_status vxm_blocklist_assign(vxm_blocklist* l, const vxm_grid_index* data, uint64_t n) {
  return guard([&] {
    l->assign_host(data, n);
  });
}

vxm_status vxm_layer_create(vxm_context* ctx, vxm_layer_type type, double vs, uint64_t max_blocks,
                            vxm_layer** out) {
  return guard([&] {
    REQUIRE_ARG(ctx && out, "null argument");
    if (!(vs > 0.0)) throw Error(VXM_ERR_INVALID_ARGUMENT, "Layer: voxel_size must be positive");
    REQUIRE_ARG(type == VXM_LAYER_TSDF || type == VXM_LAYER_ESDF || type == VXM_LAYER_OCCUPANCY ||
                    type == VXM_LAYER_COLOR,
                "unknown layer type");
    auto* L = new vxm_layer();
    L->ctx = ctx;
    L->type = type;
    L->vs = vs;
    L->max_blocks = max_blocks ? max_blocks : (uint64_t(1) << 30);
    VXM_CUDA(cudaMalloc(&L->meta, sizeof(LayerMeta)));
    // stream-ordered zeroing (the context stream does not sync with the
    // legacy stream, so a plain cudaMemset could land after the first read)
    VXM_CUDA(cudaMemsetAsync(L->meta, 0, sizeof(LayerMeta), ctx->stream));
    if (type == VXM_LAYER_ESDF) {
      // [0..2] dirty-list counts, [3..6] sweep / pair work counters by parity,
      // [7..10] round-1 split counters (zero between launches)
      VXM_CUDA(cudaMalloc(&L->dirty_count, sizeof(uint32_t) * kDirtyCountWords));
      VXM_CUDA(cudaMemsetAsync(L->dirty_count, 0, sizeof(uint32_t) * kDirtyCountWords, ctx->stream));
    }
    L->ensure_capacity(std::min<uint64_t>(4096, L->max_blocks));
    *out = L;
  });
}
void vxm_layer_destroy(vxm_layer* L) {
  if (!L) return;
  cudaStreamSynchronize(L->ctx->stream);
  delete L;
}
double vxm_layer_voxel_size(const vxm_layer* L) { return L->vs; }
vxm_status vxm_layer_reserve(vxm_layer* L, uint64_t n) {
  return guard([&] {
    REQUIRE_ARG(L, "null argument");
    L->ensure_capacity(std::min<uint64_t>(n, L->max_blocks));
  });
}
vxm_status vxm_layer_num_blocks(vxm_layer* L, uint64_t* out) {
  return guard([&] {
    L->refresh();
    *out = L->num_blocks;
  });
}
vxm_status vxm_layer_has_blocks(vxm_layer* L, const vxm_grid_index* keys, uint64_t n, uint8_t* out) {
  return guard([&] {
    std::vector<int32_t> slots;
    DevBuf ds;
    lookup_host_keys(L, keys, n, &slots, &ds);
    for (uint64_t i = 0; i < n; ++i) out[i] = slots[i] >= 0;
  });
}

vxm_status vxm_layer_export(vxm_layer* L, vxm_grid_index* keys_out, void* voxels_out,
                            uint64_t capacity) {
  return guard([&] {
    Context* ctx = L->ctx;
    std::vector<uint64_t> keys;
    std::vector<int32_t> slots;
    layer_export_sorted(L, &keys, &slots);
    const uint64_t n = keys.size();
    REQUIRE_ARG(capacity >= n, "vxm_layer_export: capacity smaller than num_blocks");
    for (uint64_t i = 0; i < n; ++i) keys_out[i] = {key_x(keys[i]), key_y(keys[i]), key_z(keys[i])};
    if (voxels_out && n) {
      const uint32_t bb = uint32_t(L->block_bytes());
      DevBuf ds, dout;
      ds.ensure(sizeof(int32_t) * n);
      dout.ensure(size_t(bb) * n);
      VXM_CUDA(cudaMemcpyAsync(ds.p, slots.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                               ctx->stream));
      k_gather_blocks<<<grid1d(ctx, n * (bb / 4)), 256, 0, ctx->stream>>>(
          static_cast<const unsigned char*>(L->cur_pool()), ds.as<int32_t>(), uint32_t(n), bb,
          dout.as<unsigned char>());
      ctx->count_launch();
      check_launch(ctx, "k_gather_blocks");
      VXM_CUDA(cudaMemcpyAsync(voxels_out, dout.p, size_t(bb) * n, cudaMemcpyDeviceToHost, ctx->stream));
      VXM_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

vxm_status vxm_layer_read_blocks(vxm_layer* L, const vxm_grid_index* keys, uint64_t n,
                                 void* voxels_out, uint8_t* found) {
  return guard([&] {
    Context* ctx = L->ctx;
    L->refresh();
    std::vector<int32_t> slots;
    DevBuf ds, dout;
    lookup_host_keys(L, keys, n, &slots, &ds);
    if (found)
      for (uint64_t i = 0; i < n; ++i) found[i] = slots[i] >= 0;
    if (!n || !voxels_out) return;
    const uint32_t bb = uint32_t(L->block_bytes());
    dout.ensure(size_t(bb) * n);
    k_gather_blocks<<<grid1d(ctx, n * (bb / 4)), 256, 0, ctx->stream>>>(
        static_cast<const unsigned char*>(L->cur_pool()), ds.as<int32_t>(), uint32_t(n), bb,
        dout.as<unsigned char>());
    ctx->count_launch();
    check_launch(ctx, "k_gather_blocks");
    VXM_CUDA(cudaMemcpyAsync(voxels_out, dout.p, size_t(bb) * n, cudaMemcpyDeviceToHost, ctx->stream));
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

vxm_status vxm_layer_write_blocks(vxm_layer* L, const vxm_grid_index* keys, uint64_t n,
                                  const void* voxels) {
  return guard([&] {
    ++L->esdf_gen;                 // (user data: breaks the ESDF quiet chain)
    L->mod_floor = next_mod_tick();  // (and, on a source layer, every mark-skip stamp)
    Context* ctx = L->ctx;
    if (!n) return;
    // last write of a duplicated key wins (sequential get_or_allocate + copy)
    std::map<std::tuple<int32_t, int32_t, int32_t>, uint64_t> last;
    for (uint64_t i = 0; i < n; ++i) last[{keys[i].x, keys[i].y, keys[i].z}] = i;
    std::vector<vxm_grid_index> uk;
    std::vector<uint64_t> src;
    for (const auto& kv : last) {
      uk.push_back({std::get<0>(kv.first), std::get<1>(kv.first), std::get<2>(kv.first)});
      src.push_back(kv.second);
    }
    L->refresh();
    vxm_blocklist list;
    list.ctx = ctx;
    list.assign_host(uk.data(), uk.size());  // already sorted + unique (std::map order)
    const uint32_t m = uint32_t(uk.size());
    DevBuf dslots;
    dslots.ensure(sizeof(int32_t) * m);
    ctx->reset_status();
    L->subset_valid = false;  // blocks not produced by mark_sites
    L->esdf_user_data = true;  // (any layer type; read for ESDF layers)
    alloc_key_list(L, &list, dslots.as<int32_t>());
    const uint32_t bb = uint32_t(L->block_bytes());
    std::vector<unsigned char> packed(size_t(bb) * m);
    for (uint32_t i = 0; i < m; ++i)
      std::memcpy(packed.data() + size_t(i) * bb, static_cast<const unsigned char*>(voxels) + src[i] * bb, bb);
    DevBuf din;
    din.ensure(packed.size());
    VXM_CUDA(cudaMemcpyAsync(din.p, packed.data(), packed.size(), cudaMemcpyHostToDevice, ctx->stream));
    k_scatter_blocks<<<grid1d(ctx, uint64_t(m) * (bb / 4)), 256, 0, ctx->stream>>>(
        static_cast<unsigned char*>(L->cur_pool()), dslots.as<int32_t>(), m, bb,
        din.as<unsigned char>());
    ctx->count_launch();
    check_launch(ctx, "k_scatter_blocks");
    if (L->site_any) {
      k_mark_site_any<<<grid1d(ctx, m), 256, 0, ctx->stream>>>(L->site_any, dslots.as<int32_t>(), m);
      ctx->count_launch();
      check_launch(ctx, "k_mark_site_any");
    }
    ctx->sync_status();
    L->refresh();
    if (ctx->h_status->capacity_error || ctx->h_status->pool_overflow)
      throw Error(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
  });
}

vxm_status vxm_layer_clone(vxm_layer* src, vxm_layer** out) {
  return guard([&] {
    src->refresh();
    const uint64_t n = src->num_blocks;
    std::vector<vxm_grid_index> keys(n);
    std::vector<unsigned char> vox(n * src->block_bytes());
    vxm_status s = vxm_layer_export(src, keys.data(), vox.data(), n);
    if (s != VXM_OK) throw Error(s, g_err);
    vxm_layer* L = nullptr;
    s = vxm_layer_create(static_cast<vxm_context*>(src->ctx), vxm_layer_type(src->type), src->vs,
                         src->max_blocks, &L);
    if (s != VXM_OK) throw Error(s, g_err);
    if (n) {
      s = vxm_layer_write_blocks(L, keys.data(), n, vox.data());
      if (s != VXM_OK) {
        vxm_layer_destroy(L);
        throw Error(s, g_err);
      }
    }
    *out = L;
  });
}

vxm_status vxm_blocks_in_view_camera(vxm_context* ctx, const vxm_pose* T, const vxm_camera* cam,
                                     const float* depth, int w, int h, double block_size,
                                     const vxm_view_config* cfg, vxm_blocklist* out) {
  return guard([&] {
    REQUIRE_ARG(ctx && T && cam && cfg && out, "null argument");
    REQUIRE_ARG(block_size > 0.0, "block_size must be positive");
    ViewArgs va{};
    va.T_LS = *T;
    va.lidar = false;
    va.cam = *cam;
    va.width = w;
    va.height = h;
    va.block_size = block_size;
    va.cfg = *cfg;
    stage_depth(ctx, depth, w, h, false, &va.depth_dev);
    ctx->reset_status();
    uint32_t cap = 0;
    run_view(ctx, va, nullptr, &cap);
    ctx->sync_status();
    if (ctx->h_status->bitmap_overflow) throw Error(VXM_ERR_INTERNAL, "candidate bitmap overflow");
    const uint32_t n = ctx->h_status->n_candidates;
    out->bind(ctx);
    out->ensure(std::max<uint32_t>(n, 1));
    VXM_CUDA(cudaMemcpyAsync(out->keys.p, ctx->cand_keys.p, sizeof(uint64_t) * n,
                             cudaMemcpyDeviceToDevice, ctx->stream));
    VXM_CUDA(cudaMemcpyAsync(out->d_count, &ctx->d_status->n_candidates, sizeof(uint32_t),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    out->host_valid = false;
    out->host_pending = false;
    out->count_hint = n;
    out->sorted_unique = true;
    out->fetch();
  });
}

vxm_status vxm_blocks_in_view_lidar(vxm_context* ctx, const vxm_pose* T, const vxm_lidar* li,
                                    const float* depth, int w, int h, double block_size,
                                    const vxm_view_config* cfg, vxm_blocklist* out) {
  return guard([&] {
    REQUIRE_ARG(ctx && T && li && cfg && out, "null argument");
    REQUIRE_ARG(block_size > 0.0, "block_size must be positive");
    REQUIRE_ARG(w == li->num_azimuth && h == li->num_elevation,
                "blocks_in_view: image size does not match intrinsics");
    ViewArgs va{};
    va.T_LS = *T;
    va.lidar = true;
    va.li = *li;
    va.width = w;
    va.height = h;
    va.block_size = block_size;
    va.cfg = *cfg;
    stage_depth(ctx, depth, w, h, false, &va.depth_dev);
    ctx->reset_status();
    uint32_t cap = 0;
    run_view(ctx, va, nullptr, &cap);
    ctx->sync_status();
    if (ctx->h_status->bitmap_overflow) throw Error(VXM_ERR_INTERNAL, "candidate bitmap overflow");
    const uint32_t n = ctx->h_status->n_candidates;
    out->bind(ctx);
    out->ensure(std::max<uint32_t>(n, 1));
    VXM_CUDA(cudaMemcpyAsync(out->keys.p, ctx->cand_keys.p, sizeof(uint64_t) * n,
                             cudaMemcpyDeviceToDevice, ctx->stream));
    VXM_CUDA(cudaMemcpyAsync(out->d_count, &ctx->d_status->n_candidates, sizeof(uint32_t),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    out->host_valid = false;
    out->host_pending = false;
    out->count_hint = n;
    out->sorted_unique = true;
    out->fetch();
  });
}

vxm_status vxm_integrate_depth_camera(vxm_layer* L, const float* depth, int w, int h,
                                      const vxm_pose* T, const vxm_camera* cam,
                                      const vxm_integrator_config* cfg, vxm_blocklist* out) {
  return integrate_common(L, depth, w, h, T, cam, nullptr, cfg, out, false);
}
vxm_status vxm_integrate_depth_lidar(vxm_layer* L, const float* depth, int w, int h,
                                     const vxm_pose* T, const vxm_lidar* li,
                                     const vxm_integrator_config* cfg, vxm_blocklist* out) {
  return integrate_common(L, depth, w, h, T, nullptr, li, cfg, out, false);
}
vxm_status vxm_integrate_depth_camera_device(vxm_layer* L, const float* depth, int w, int h,
                                             const vxm_pose* T, const vxm_camera* cam,
                                             const vxm_integrator_config* cfg, vxm_blocklist* out) {
  return integrate_common(L, depth, w, h, T, cam, nullptr, cfg, out, true);
}
vxm_status vxm_integrate_depth_lidar_device(vxm_layer* L, const float* depth, int w, int h,
                                            const vxm_pose* T, const vxm_lidar* li,
                                            const vxm_integrator_config* cfg, vxm_blocklist* out) {
  return integrate_common(L, depth, w, h, T, nullptr, li, cfg, out, true);
}

vxm_status vxm_update_frame_camera_device(vxm_layer* T, vxm_layer* E, const float* depth, int w,
                                          int h, const vxm_pose* pose, const vxm_camera* cam,
                                          const vxm_integrator_config* icfg,
                                          const vxm_esdf_config* ecfg, vxm_blocklist* tout,
                                          vxm_blocklist* eout) {
  return frame_common(T, E, depth, w, h, pose, cam, nullptr, icfg, ecfg, tout, eout);
}
vxm_status vxm_update_frame_lidar_device(vxm_layer* T, vxm_layer* E, const float* depth, int w,
                                         int h, const vxm_pose* pose, const vxm_lidar* li,
                                         const vxm_integrator_config* icfg,
                                         const vxm_esdf_config* ecfg, vxm_blocklist* tout,
                                         vxm_blocklist* eout) {
  return frame_common(T, E, depth, w, h, pose, nullptr, li, icfg, ecfg, tout, eout);
}

vxm_status vxm_update_esdf_sharded(int P, vxm_layer* const* esdf, vxm_layer* const* tsdf,
                                   vxm_blocklist* const* updated, const vxm_esdf_config* cfg,
                                   vxm_blocklist* const* out) {
  return guard([&] {
    REQUIRE_ARG(P >= 1 && esdf && tsdf && updated && cfg && out, "null argument");
    std::vector<Layer*> E(P), T(P);
    std::vector<BlockList*> U(P), O(P);
    int slab = 0;
    for (int p = 0; p < P; ++p) {
      REQUIRE_ARG(esdf[p] && tsdf[p] && updated[p] && out[p], "null argument");
      REQUIRE_ARG(esdf[p]->type == VXM_LAYER_ESDF && tsdf[p]->type == VXM_LAYER_TSDF,
                  "update_esdf: expects (ESDF layer, TSDF layer)");
      Context* ctx = esdf[p]->ctx;
      REQUIRE_ARG(tsdf[p]->ctx == ctx, "update_esdf_sharded: shard layers on different contexts");
      REQUIRE_ARG(ctx->world == P && ctx->rank == p,
                  "update_esdf_sharded: shard p's context must be set_shard(p, n_shards, slab)");
      if (p == 0) slab = ctx->slab;
      REQUIRE_ARG(ctx->slab == slab, "update_esdf_sharded: shards disagree on the slab width");
      for (int q = 0; q < p; ++q)
        REQUIRE_ARG(esdf[q]->ctx != ctx, "update_esdf_sharded: one context per shard");
      if (esdf[p]->vs != tsdf[p]->vs || esdf[p]->vs != esdf[0]->vs)
        throw Error(VXM_ERR_INVALID_ARGUMENT, "update_esdf: source and ESDF layer voxel sizes differ");
      ensure_sorted_unique(updated[p]);
      E[p] = esdf[p];
      T[p] = tsdf[p];
      U[p] = updated[p];
      O[p] = out[p];
    }
    run_update_esdf_sharded(P, E.data(), T.data(), U.data(), *cfg, slab, O.data());
  });
}

struct vxm_shard_update {
  vxm::ShardUpdate x;
};

vxm_status vxm_shard_update_begin(vxm_layer* E, vxm_layer* T, vxm_blocklist* uni,
                                  const vxm_esdf_config* cfg, vxm_shard_update** out, int* any) {
  vxm_shard_update* su = nullptr;
  const vxm_status st = guard([&] {
    REQUIRE_ARG(E && T && uni && cfg && out && any, "null argument");
    REQUIRE_ARG(E->type == VXM_LAYER_ESDF && T->type == VXM_LAYER_TSDF,
                "update_esdf: expects (ESDF layer, TSDF layer)");
    REQUIRE_ARG(E->ctx == T->ctx && uni->ctx == E->ctx, "shard update: objects on different contexts");
    if (E->vs != T->vs)
      throw Error(VXM_ERR_INVALID_ARGUMENT, "update_esdf: source and ESDF layer voxel sizes differ");
    su = new vxm_shard_update();
    ShardUpdate& x = su->x;
    x.E = E;
    x.T = T;
    x.ctx = E->ctx;
    x.rank = x.ctx->rank;
    x.world = x.ctx->world;
    x.slab = x.ctx->slab;
    ensure_sorted_unique(uni);
    // a private copy of the union (the caller's list may be reused)
    x.uni.ctx = x.ctx;
    const uint32_t n = std::max<uint32_t>(uni->count_hint, 1);
    x.uni.ensure(n);
    VXM_CUDA(cudaMemcpyAsync(x.uni.keys.p, uni->keys.p, sizeof(uint64_t) * uni->count_hint,
                             cudaMemcpyDeviceToDevice, x.ctx->stream));
    VXM_CUDA(cudaMemcpyAsync(x.uni.d_count, uni->d_count, sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                             x.ctx->stream));
    x.uni.count_hint = uni->count_hint;
    x.uni.host_valid = false;
    x.uni.host_pending = false;
    x.uni.sorted_unique = true;
    shard_begin(x, *cfg);
    *any = x.local_any ? 1 : 0;
    *out = su;
  });
  if (st != VXM_OK) delete su;
  return st;
}
vxm_status vxm_shard_update_plan(vxm_shard_update* su, uint32_t* n) {
  return guard([&] {
    REQUIRE_ARG(su && n, "null argument");
    shard_plan(su->x);
    *n = su->x.n_bnd;
  });
}
vxm_status vxm_shard_update_exchange_buffers(vxm_shard_update* su, uint32_t n_left, uint32_t n_right,
                                             void** send, uint64_t* send_bytes, void** recv_left,
                                             uint64_t* recv_left_bytes, void** recv_right,
                                             uint64_t* recv_right_bytes) {
  return guard([&] {
    REQUIRE_ARG(su && send && send_bytes && recv_left && recv_left_bytes && recv_right && recv_right_bytes,
                "null argument");
    shard_set_neighbours(su->x, n_left, n_right);
    *send = su->x.snd.p;
    *send_bytes = xbuf_bytes(su->x.n_bnd);
    *recv_left = su->x.rcv[0].p;
    *recv_left_bytes = xbuf_bytes(n_left);
    *recv_right = su->x.rcv[1].p;
    *recv_right_bytes = xbuf_bytes(n_right);
  });
}
vxm_status vxm_shard_update_sweep(vxm_shard_update* su, uint32_t round) {
  return guard([&] {
    REQUIRE_ARG(su && round >= 1, "invalid argument");
    shard_sweep(su->x, round);
  });
}
vxm_status vxm_shard_update_border(vxm_shard_update* su, uint32_t round, uint32_t* next) {
  return guard([&] {
    REQUIRE_ARG(su && round >= 1, "invalid argument");
    if (next)
      *next = shard_border(su->x, round);
    else
      shard_border_launch(su->x, round);
  });
}
vxm_status vxm_shard_update_ipc_handles(vxm_shard_update* su, void* handles_out) {
  return guard([&] {
    REQUIRE_ARG(su && handles_out, "null argument");
    shard_ipc_handles(su->x, handles_out);
  });
}
vxm_status vxm_shard_update_lower_fused(vxm_shard_update* su, const void* all_handles, int ranks_on_device) {
  return guard([&] {
    REQUIRE_ARG(su && all_handles && ranks_on_device >= 1, "invalid argument");
    shard_lower_fused_ipc(su->x, all_handles, ranks_on_device);
  });
}
vxm_status vxm_shard_update_next_count(vxm_shard_update* su, uint32_t round, void** dptr) {
  return guard([&] {
    REQUIRE_ARG(su && dptr && round >= 1, "invalid argument");
    *dptr = next_count_ptr(su->x, round);
  });
}
vxm_status vxm_shard_update_finish(vxm_shard_update* su, int lowered, vxm_blocklist* out) {
  const vxm_status st = guard([&] {
    REQUIRE_ARG(su && out, "null argument");
    shard_finish(su->x, lowered != 0, out);
  });
  delete su;
  return st;
}
void vxm_shard_update_destroy(vxm_shard_update* su) { delete su; }

vxm_status vxm_update_esdf_list(vxm_layer* E, vxm_layer* T, vxm_blocklist* updated,
                                const vxm_esdf_config* cfg, vxm_blocklist* out) {
  return guard([&] {
    REQUIRE_ARG(E && T && updated && cfg && out, "null argument");
    REQUIRE_ARG(E->type == VXM_LAYER_ESDF && is_source(T),
                "update_esdf: expects (ESDF layer, TSDF or occupancy layer)");
    out->bind(E->ctx);
    // esdf/integrator.cpp:371-378: empty input returns {} before the size check
    if (updated->count_hint == 0 || (updated->host_valid && updated->host.empty())) {
      out->assign_host(nullptr, 0);
      out->sorted_unique = true;
      return;
    }
    if (E->vs != T->vs)
      throw Error(VXM_ERR_INVALID_ARGUMENT, "update_esdf: source and ESDF layer voxel sizes differ");
    ensure_sorted_unique(updated);
    run_update_esdf(E, T, updated, *cfg, out);
    out->sorted_unique = true;
  });
}

vxm_status vxm_update_esdf(vxm_layer* E, vxm_layer* T, const vxm_grid_index* updated, uint64_t n,
                           const vxm_esdf_config* cfg, vxm_blocklist* out) {
  return guard([&] {
    REQUIRE_ARG(E && T && cfg && out, "null argument");
    Context* ctx = E->ctx;
    if (!ctx->scratch_in) {  // reused input list: no per-call device allocations
      ctx->scratch_in = new vxm_blocklist();
      ctx->scratch_in->ctx = ctx;
    }
    HostTrace tr("update_esdf");
    tr.dev_mark(ctx->stream, "start");
    vxm_blocklist* list = static_cast<vxm_blocklist*>(ctx->scratch_in);
    BlockList* last = ctx->last_host_out;
    if (last && last != out && last->ctx == ctx && last->host_valid && last->sorted_unique && last->host.size() == n &&
        (n == 0 || std::memcmp(last->host.data(), updated, sizeof(vxm_grid_index) * n) == 0)) {
      list = static_cast<vxm_blocklist*>(last);  // the integrate's device keys, identical content
    } else {
      list->assign_host(updated, n, false);  // (an input only: no host copy)
    }
    tr.mark("assigned");
    tr.dev_mark(ctx->stream, "h2d");
    out->want_host = true;  // unpacked to mapped host memory before the one sync
    const vxm_status s = vxm_update_esdf_list(E, T, list, cfg, out);
    out->want_host = false;
    if (s != VXM_OK) throw Error(s, g_err);
    tr.mark("synced");
    out->fetch();
    tr.mark("fetched");
  });
}

vxm_status vxm_esdf_state_create(vxm_esdf_state** out) {
  return guard([&] { *out = new vxm_esdf_state(); });
}
void vxm_esdf_state_destroy(vxm_esdf_state* st) { delete st; }
vxm_status vxm_esdf_state_get(vxm_esdf_state* st, int which, const vxm_grid_index** data,
                              uint64_t* n) {
  return guard([&] {
    REQUIRE_ARG(which >= 0 && which < 3, "state list index");
    *data = st->lists[which].data();
    *n = st->lists[which].size();
  });
}
vxm_status vxm_esdf_state_set(vxm_esdf_state* st, int which, const vxm_grid_index* data, uint64_t n) {
  return guard([&] {
    REQUIRE_ARG(which >= 0 && which < 3, "state list index");
    st->lists[which].assign(data, data + n);
  });
}

vxm_status vxm_esdf_mark_sites(vxm_layer* E, vxm_layer* T, const vxm_grid_index* updated, uint64_t n,
                               const vxm_esdf_config* cfg, vxm_esdf_state* st,
                               vxm_blocklist* changed) {
  return guard([&] {
    REQUIRE_ARG(E && T && cfg && st && changed, "null argument");
    REQUIRE_ARG(E->type == VXM_LAYER_ESDF && is_source(T),
                "mark_sites: expects (ESDF layer, TSDF or occupancy layer)");
    std::vector<vxm_grid_index> ch;
    if (n) {
      vxm_blocklist list;
      list.ctx = E->ctx;
      list.assign_host(updated, n);
      ensure_sorted_unique(&list);
      run_mark_sites(E, T, &list, *cfg, st, &ch);
    }
    changed->bind(E->ctx);
    changed->assign_host(ch.data(), ch.size());
  });
}
vxm_status vxm_esdf_clear_invalid(vxm_layer* E, const vxm_esdf_config* cfg, vxm_esdf_state* st,
                                  vxm_blocklist* changed) {
  return guard([&] {
    std::vector<vxm_grid_index> ch;
    run_clear_invalid(E, *cfg, st, &ch);
    changed->bind(E->ctx);
    changed->assign_host(ch.data(), ch.size());
  });
}
vxm_status vxm_esdf_lower(vxm_layer* E, vxm_esdf_state* st, const vxm_esdf_config* cfg,
                          vxm_blocklist* changed, int* rounds) {
  return guard([&] {
    std::vector<vxm_grid_index> ch;
    const int r = run_lower_esdf(E, st, *cfg, &ch);
    if (rounds) *rounds = r;
    changed->bind(E->ctx);
    changed->assign_host(ch.data(), ch.size());
  });
}

vxm_status vxm_query_batch(vxm_layer* E, const double* xyz, uint64_t n, int want_gradient,
                           const vxm_query_config* cfg, vxm_query_result* out) {
  return guard([&] {
    REQUIRE_ARG(E && cfg && (n == 0 || (xyz && out)), "null argument");
    REQUIRE_ARG(E->type == VXM_LAYER_ESDF, "query_batch: expects an ESDF layer");
    run_query(E, xyz, n, want_gradient, cfg->interpolate, out);
  });
}

}  // extern "C"

// ---- VXLF snapshots — core/serialization.cpp:20-158 (format: FORMATS.md) ------
namespace {
constexpr char kVxlfMagic[4] = {'V', 'X', 'L', 'F'};
constexpr uint32_t kVxlfVersion = 1;

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};
void io_fail(const std::string& m) { throw Error(VXM_ERR_IO, m); }
template <typename T>
void put(FILE* f, const T& v) {
  if (std::fwrite(&v, sizeof(T), 1, f) != 1) io_fail("snapshot: write failed");
}
template <typename T>
void get(FILE* f, T* v) {
  if (std::fread(v, sizeof(T), 1, f) != 1) io_fail("snapshot: truncated file");
}

// write_layer — serialization.cpp:42-60: name, voxel bytes, count, then per
// block (x, y, z) and the voxel payload, in sorted order.  The device gathers
// the sorted blocks (vxm_layer_export); records are streamed in chunks.
void write_layer(FILE* f, const char* name, vxm_layer* L) {
  const uint32_t name_len = uint32_t(std::strlen(name));
  put(f, name_len);
  if (std::fwrite(name, 1, name_len, f) != name_len) io_fail("snapshot: write failed");
  const uint32_t vb = uint32_t(L->voxel_bytes());
  put(f, vb);
  L->refresh();
  const uint64_t n = L->num_blocks;
  put(f, n);
  std::vector<vxm_grid_index> keys(n);
  std::vector<unsigned char> vox(n * L->block_bytes());
  vxm_status st = vxm_layer_export(L, keys.data(), vox.data(), n);
  if (st != VXM_OK) throw Error(st, g_err);
  const size_t bb = L->block_bytes();
  for (uint64_t i = 0; i < n; ++i) {
    put(f, keys[i].x);
    put(f, keys[i].y);
    put(f, keys[i].z);
    if (std::fwrite(vox.data() + i * bb, 1, bb, f) != bb) io_fail("snapshot: write failed");
  }
}

// read_layer — serialization.cpp:62-82
void read_layer(FILE* f, vxm_layer* L) {
  uint32_t vb = 0;
  get(f, &vb);
  if (vb != L->voxel_bytes()) io_fail("snapshot: voxel size mismatch for layer payload");
  uint64_t n = 0;
  get(f, &n);
  const size_t bb = L->block_bytes();
  std::vector<vxm_grid_index> keys;
  std::vector<unsigned char> vox;
  for (uint64_t i = 0; i < n; ++i) {
    vxm_grid_index g;
    get(f, &g.x);
    get(f, &g.y);
    get(f, &g.z);
    keys.push_back(g);
    vox.resize(keys.size() * bb);
    if (std::fread(vox.data() + (keys.size() - 1) * bb, 1, bb, f) != bb)
      io_fail("snapshot: truncated block payload");
  }
  if (!keys.empty()) {
    const vxm_status st = vxm_layer_write_blocks(L, keys.data(), keys.size(), vox.data());
    if (st != VXM_OK) throw Error(st, g_err);
  }
}
}  // namespace

extern "C" {
vxm_status vxm_snapshot_save_layers(const char* path, double vs, vxm_layer* tsdf, vxm_layer* occ,
                                    vxm_layer* color, vxm_layer* esdf) {
  return guard([&] {
    REQUIRE_ARG(path, "null argument");
    REQUIRE_ARG(!tsdf || tsdf->type == VXM_LAYER_TSDF, "snapshot: tsdf argument is not a TSDF layer");
    REQUIRE_ARG(!occ || occ->type == VXM_LAYER_OCCUPANCY,
                "snapshot: occupancy argument is not an occupancy layer");
    REQUIRE_ARG(!color || color->type == VXM_LAYER_COLOR, "snapshot: color argument is not a color layer");
    REQUIRE_ARG(!esdf || esdf->type == VXM_LAYER_ESDF, "snapshot: esdf argument is not an ESDF layer");
    REQUIRE_ARG((!tsdf || tsdf->vs == vs) && (!occ || occ->vs == vs) && (!color || color->vs == vs) &&
                    (!esdf || esdf->vs == vs),
                "snapshot: layer voxel size differs from the snapshot's");
    File out;
    out.f = std::fopen(path, "wb");
    if (!out.f) io_fail(std::string("snapshot: cannot open for writing: ") + path);
    if (std::fwrite(kVxlfMagic, 1, 4, out.f) != 4) io_fail("snapshot: write failed");
    put(out.f, kVxlfVersion);
    put(out.f, vs);  // f64
    const uint32_t count = (tsdf ? 1u : 0u) + (occ ? 1u : 0u) + (color ? 1u : 0u) + (esdf ? 1u : 0u);
    put(out.f, count);
    if (tsdf) write_layer(out.f, "tsdf", tsdf);  // serialization.cpp:102-105 order
    if (occ) write_layer(out.f, "occupancy", occ);
    if (color) write_layer(out.f, "color", color);
    if (esdf) write_layer(out.f, "esdf", esdf);
    if (std::fflush(out.f) != 0) io_fail(std::string("snapshot: write failed: ") + path);
  });
}
vxm_status vxm_snapshot_save(const char* path, double vs, vxm_layer* tsdf, vxm_layer* esdf) {
  return vxm_snapshot_save_layers(path, vs, tsdf, nullptr, nullptr, esdf);
}

vxm_status vxm_snapshot_load_layers(vxm_context* ctx, const char* path, double* vs_out,
                                    vxm_layer** tsdf_out, vxm_layer** occ_out, vxm_layer** color_out,
                                    vxm_layer** esdf_out) {
  vxm_layer* T = nullptr;
  vxm_layer* O = nullptr;
  vxm_layer* Cl = nullptr;
  vxm_layer* E = nullptr;
  const vxm_status st = guard([&] {
    REQUIRE_ARG(ctx && path && tsdf_out && esdf_out, "null argument");
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) io_fail(std::string("snapshot: cannot open: ") + path);
    char magic[4];
    if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, kVxlfMagic, 4) != 0)
      io_fail("snapshot: bad magic");
    uint32_t version = 0;
    get(in.f, &version);
    if (version != kVxlfVersion) io_fail("snapshot: unsupported version " + std::to_string(version));
    double vs = 0.0;
    get(in.f, &vs);
    if (!(vs > 0.0)) io_fail("snapshot: invalid voxel size");
    uint32_t count = 0;
    get(in.f, &count);
    for (uint32_t i = 0; i < count; ++i) {
      uint32_t name_len = 0;
      get(in.f, &name_len);
      if (name_len > 64) io_fail("snapshot: layer name too long");
      std::string name(name_len, '\0');
      if (std::fread(name.data(), 1, name_len, in.f) != name_len) io_fail("snapshot: truncated layer name");
      if (name == "tsdf" || name == "esdf" || (name == "occupancy" && occ_out) ||
          (name == "color" && color_out)) {
        vxm_layer*& L = name == "tsdf" ? T : name == "esdf" ? E : name == "color" ? Cl : O;
        if (!L) {
          const vxm_layer_type type = name == "tsdf"    ? VXM_LAYER_TSDF
                                      : name == "esdf"  ? VXM_LAYER_ESDF
                                      : name == "color" ? VXM_LAYER_COLOR
                                                        : VXM_LAYER_OCCUPANCY;
          const vxm_status s = vxm_layer_create(ctx, type, vs, 0, &L);
          if (s != VXM_OK) throw Error(s, g_err);
        }
        read_layer(in.f, L);
      } else if (name == "occupancy" || name == "color") {
        io_fail("snapshot: the file holds a" + std::string(name == "occupancy" ? "n " : " ") + name +
                " layer (use vxm_snapshot_load_layers)");
      } else {
        io_fail("snapshot: unknown layer name '" + name + "'");
      }
    }
    *vs_out = vs;
    *tsdf_out = T;
    if (occ_out) *occ_out = O;
    if (color_out) *color_out = Cl;
    *esdf_out = E;
  });
  if (st != VXM_OK) {
    vxm_layer_destroy(T);
    vxm_layer_destroy(O);
    vxm_layer_destroy(Cl);
    vxm_layer_destroy(E);
  }
  return st;
}
vxm_status vxm_snapshot_load(vxm_context* ctx, const char* path, double* vs_out, vxm_layer** tsdf_out,
                             vxm_layer** esdf_out) {
  return vxm_snapshot_load_layers(ctx, path, vs_out, tsdf_out, nullptr, nullptr, esdf_out);
}
}  // extern "C"

// ---- replay — io/pipeline.cpp:46-148 --------------------------------------------
namespace {
double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

vxm_status replay_common(vxm_context* ctx, const vxm_replay_config* cfg, const vxm_camera* cam,
                         const vxm_lidar* li, int n, int w, int h, const float* depth,
                         const uint8_t* rgb, const vxm_pose* poses, vxm_replay_result* res,
                         vxm_frame_timing* timings) {
  vxm_layer* T = nullptr;
  vxm_layer* E = nullptr;
  vxm_layer* Cl = nullptr;
  vxm_mesh_layer* M = nullptr;
  const vxm_status st = guard([&] {
    REQUIRE_ARG(ctx && cfg && (cam || li) && res && timings, "null argument");
    if (n <= 0) throw Error(VXM_ERR_INVALID_ARGUMENT, "replay: dataset has no frames");
    if (cfg->update_every < 1) throw Error(VXM_ERR_INVALID_ARGUMENT, "replay: update_every must be >= 1");
    if (cfg->with_color && (cfg->use_occupancy || !cam))
      throw Error(VXM_ERR_INVALID_ARGUMENT, "replay: color needs a camera dataset fused into a TSDF map");
    REQUIRE_ARG(depth && poses, "null argument");
    // the source layer: TSDF, or occupancy with use_occupancy (pipeline.cpp:95-101)
    vxm_status s = vxm_layer_create(ctx, cfg->use_occupancy ? VXM_LAYER_OCCUPANCY : VXM_LAYER_TSDF,
                                    cfg->voxel_size, 0, &T);
    if (s != VXM_OK) throw Error(s, g_err);
    vxm_blocklist changed, esdf_changed, pending, color_changed;
    changed.ctx = esdf_changed.ctx = pending.ctx = color_changed.ctx = ctx;
    uint32_t n_pending = 0;  // keys in `pending` (unsorted, may repeat until folded)
    DevBuf grow;
    const size_t frame_px = size_t(w) * size_t(h);
    for (int k = 0; k < n; ++k) {
      vxm_frame_timing& t = timings[k];
      t = vxm_frame_timing{k, 0.0, 0.0, 0.0, 0.0};
      const auto t0 = std::chrono::steady_clock::now();
      const ViewArgs va = frame_args(T, depth + size_t(k) * frame_px, w, h, &poses[k], cam, li,
                                     &cfg->integrator, false);
      run_integrate(T, va, cfg->integrator, &changed);
      t.tsdf_ms = ms_since(t0);
      // pending ∪= changed (pipeline.cpp:38-43; folded with one sort at the update)
      const uint32_t n_ch = ctx->h_status->n_changed;
      if (n_ch) {
        if (n_pending + n_ch > pending.cap) {
          const uint32_t cap = std::max<uint32_t>(2 * (n_pending + n_ch), 4096);
          grow.ensure(sizeof(uint64_t) * cap);
          if (n_pending)
            VXM_CUDA(cudaMemcpyAsync(grow.p, pending.keys.p, sizeof(uint64_t) * n_pending,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
          pending.ensure(cap);
          if (n_pending)
            VXM_CUDA(cudaMemcpyAsync(pending.keys.p, grow.p, sizeof(uint64_t) * n_pending,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
        }
        VXM_CUDA(cudaMemcpyAsync(pending.keys.as<uint64_t>() + n_pending, changed.keys.p,
                                 sizeof(uint64_t) * n_ch, cudaMemcpyDeviceToDevice, ctx->stream));
        n_pending += n_ch;
      }
      if (cfg->with_color && rgb) {  // pipeline.cpp:111-117
        const auto tc = std::chrono::steady_clock::now();
        if (!Cl) {
          s = vxm_layer_create(ctx, VXM_LAYER_COLOR, cfg->voxel_size, 0, &Cl);
          if (s != VXM_OK) throw Error(s, g_err);
        }
        const ViewArgs vc = frame_args(T, depth + size_t(k) * frame_px, w, h, &poses[k], cam, nullptr,
                                       &cfg->integrator, false);
        run_integrate_color(Cl, T, rgb + size_t(k) * frame_px * 3, vc, cfg->integrator, &color_changed);
        t.color_ms = ms_since(tc);
      }
      const bool last = k + 1 == n;
      const bool on_cadence = (k + 1) % cfg->update_every == 0;
      if ((on_cadence || last) && n_pending > 0) {  // derive_layers (pipeline.cpp:71-86)
        const auto t1 = std::chrono::steady_clock::now();
        if (!E) {
          s = vxm_layer_create(ctx, VXM_LAYER_ESDF, cfg->voxel_size, 0, &E);
          if (s != VXM_OK) throw Error(s, g_err);
        }
        VXM_CUDA(cudaMemcpyAsync(pending.d_count, &n_pending, sizeof n_pending, cudaMemcpyHostToDevice,
                                 ctx->stream));
        pending.count_hint = n_pending;
        pending.host_valid = false;
        pending.host_pending = false;
        pending.sorted_unique = false;
        sort_unique_keys(ctx, &pending);
        pending.sorted_unique = true;
        run_update_esdf(E, T, &pending, cfg->esdf, &esdf_changed);
        t.esdf_ms = ms_since(t1);
        if (!cfg->use_occupancy) {
          const auto t2 = std::chrono::steady_clock::now();
          if (!M) {
            s = vxm_mesh_layer_create(ctx, cfg->voxel_size, &M);
            if (s != VXM_OK) throw Error(s, g_err);
          }
          run_update_mesh(M, T, &pending, cfg->mesh.min_weight, Cl);
          t.mesh_ms = ms_since(t2);
        }
        n_pending = 0;
      }
    }
    *res = vxm_replay_result{T, E, Cl, M};
  });
  if (st != VXM_OK) {
    vxm_layer_destroy(T);
    vxm_layer_destroy(E);
    vxm_layer_destroy(Cl);
    vxm_mesh_layer_destroy(M);
  }
  return st;
}
}  // namespace

extern "C" {
void vxm_replay_config_make(double voxel_size, vxm_replay_config* out) {
  out->voxel_size = voxel_size;
  out->update_every = 4;
  out->use_occupancy = 0;
  out->with_color = 0;
  vxm_mesh_config_default(&out->mesh);
  vxm_integrator_config_default(&out->integrator);
  vxm_esdf_config_default(&out->esdf);
  out->integrator.truncation = 4.0 * voxel_size;
  out->esdf.site_threshold = voxel_size;
}
vxm_status vxm_replay_camera(vxm_context* ctx, const vxm_replay_config* cfg, const vxm_camera* cam,
                             int n, int w, int h, const float* depth, const uint8_t* rgb,
                             const vxm_pose* poses, vxm_replay_result* out, vxm_frame_timing* timings) {
  return replay_common(ctx, cfg, cam, nullptr, n, w, h, depth, rgb, poses, out, timings);
}
vxm_status vxm_replay_lidar(vxm_context* ctx, const vxm_replay_config* cfg, const vxm_lidar* li, int n,
                            int w, int h, const float* depth, const vxm_pose* poses,
                            vxm_replay_result* out, vxm_frame_timing* timings) {
  return replay_common(ctx, cfg, nullptr, li, n, w, h, depth, nullptr, poses, out, timings);
}
}  // extern "C"

// ---- color fusion + meshing + PLY -----------------------

namespace {
// save_mesh_ply — ply.cpp:33-105: header, vertices (x y z nx ny nz [r g b]) of
// the non-empty blocks in sorted order, then faces with global indices.
void write_ply(const MeshLayerH& M, const char* path) {
  uint64_t nv = 0, nf = 0;
  bool with_color = true;
  for (const auto& kv : M.blocks) {
    const MeshBlockH& b = kv.second;
    if (b.triangles.empty()) continue;
    nv += b.vertices.size() / 3;
    nf += b.triangles.size() / 3;
    with_color = with_color && b.colors.size() == b.vertices.size();
  }
  if (nv == 0) with_color = false;
  File out;
  out.f = std::fopen(path, "wb");
  if (!out.f) io_fail(std::string("cannot open for writing: ") + path);
  std::string hdr = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(nv) +
                    "\nproperty float x\nproperty float y\nproperty float z\n"
                    "property float nx\nproperty float ny\nproperty float nz\n";
  if (with_color) hdr += "property uchar red\nproperty uchar green\nproperty uchar blue\n";
  hdr += "element face " + std::to_string(nf) + "\nproperty list uchar int vertex_indices\nend_header\n";
  std::vector<unsigned char> buf(hdr.begin(), hdr.end());
  auto raw = [&buf](const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    buf.insert(buf.end(), c, c + n);
  };
  for (const auto& kv : M.blocks) {
    const MeshBlockH& b = kv.second;
    if (b.triangles.empty()) continue;
    const size_t n = b.vertices.size() / 3;
    for (size_t i = 0; i < n; ++i) {
      raw(&b.vertices[3 * i], 12);
      raw(&b.normals[3 * i], 12);
      if (with_color) raw(&b.colors[3 * i], 3);
    }
  }
  uint32_t offset = 0;
  for (const auto& kv : M.blocks) {
    const MeshBlockH& b = kv.second;
    if (b.triangles.empty()) continue;
    for (size_t t = 0; t < b.triangles.size(); t += 3) {
      const unsigned char three = 3;
      raw(&three, 1);
      for (int k = 0; k < 3; ++k) {
        const int32_t v = int32_t(b.triangles[t + k] + offset);
        raw(&v, 4);
      }
    }
    offset += uint32_t(b.vertices.size() / 3);
  }
  if (std::fwrite(buf.data(), 1, buf.size(), out.f) != buf.size() || std::fflush(out.f) != 0)
    io_fail(std::string("failed while writing: ") + path);
}
}  // namespace

extern "C" {
vxm_status vxm_integrate_color(vxm_layer* C, const uint8_t* rgb, int w, int h, const float* depth,
                               int dw, int dh, const vxm_pose* T, const vxm_camera* cam,
                               vxm_layer* tsdf, const vxm_integrator_config* cfg, vxm_blocklist* out) {
  return guard([&] {
    REQUIRE_ARG(C && T && cam && tsdf && cfg && out, "integrate_color: null argument");
    REQUIRE_ARG(C->type == VXM_LAYER_COLOR, "integrate_color: layer is not a color layer");
    REQUIRE_ARG(tsdf->type == VXM_LAYER_TSDF, "integrate_color: source is not a TSDF layer");
    REQUIRE_ARG(C->ctx == tsdf->ctx, "integrate_color: layers on different contexts");
    check_pose(T);  // check_frame — integrator.cpp:26-34, 198
    if (w != cam->width || h != cam->height)
      throw Error(VXM_ERR_INVALID_ARGUMENT, "integrate: image size does not match intrinsics");
    if (dw != cam->width || dh != cam->height)
      throw Error(VXM_ERR_INVALID_ARGUMENT, "integrate_color: depth size mismatch");
    REQUIRE_ARG(w == 0 || h == 0 || (rgb && depth), "integrate_color: null image");
    ViewArgs va{};
    va.T_LS = *T;
    va.lidar = false;
    va.cam = *cam;
    va.width = w;
    va.height = h;
    va.block_size = C->vs * kVPS;
    va.cfg = {cfg->max_integration_distance, cfg->truncation, cfg->view_pixel_subsample};
    stage_depth(C->ctx, depth, w, h, false, &va.depth_dev);
    out->bind(C->ctx);
    run_integrate_color(C, tsdf, rgb, va, *cfg, out);
  });
}

void vxm_mesh_config_default(vxm_mesh_config* c) {
  c->min_weight = 1e-4f;  // marching_cubes.hpp:27
  c->parallel = 1;
}
vxm_status vxm_mesh_layer_create(vxm_context* ctx, double vs, vxm_mesh_layer** out) {
  return guard([&] {
    REQUIRE_ARG(ctx && out, "null argument");
    auto* m = new vxm_mesh_layer();
    m->ctx = ctx;
    m->vs = vs;
    *out = m;
  });
}
void vxm_mesh_layer_destroy(vxm_mesh_layer* m) { delete m; }
double vxm_mesh_layer_voxel_size(const vxm_mesh_layer* m) { return m->vs; }
uint64_t vxm_mesh_layer_num_blocks(const vxm_mesh_layer* m) { return m ? m->blocks.size() : 0; }
vxm_status vxm_mesh_layer_sorted_indices(const vxm_mesh_layer* m, vxm_grid_index* keys, uint64_t cap) {
  return guard([&] {
    REQUIRE_ARG(m && (keys || m->blocks.empty()), "null argument");
    REQUIRE_ARG(cap >= m->blocks.size(), "mesh sorted_indices: capacity smaller than num_blocks");
    uint64_t i = 0;
    for (const auto& kv : m->blocks) keys[i++] = {key_x(kv.first), key_y(kv.first), key_z(kv.first)};
  });
}
vxm_status vxm_mesh_layer_block(const vxm_mesh_layer* m, const vxm_grid_index* g, vxm_mesh_block_view* out,
                                int* found) {
  return guard([&] {
    REQUIRE_ARG(m && g && out && found, "null argument");
    *out = vxm_mesh_block_view{};
    *found = 0;
    if (!(coord_ok(g->x) && coord_ok(g->y) && coord_ok(g->z))) return;
    const auto it = m->blocks.find(pack_key(g->x, g->y, g->z));
    if (it == m->blocks.end()) return;
    const MeshBlockH& b = it->second;
    *found = 1;
    out->n_vertices = b.vertices.size() / 3;
    out->n_triangles = b.triangles.size() / 3;
    out->n_colors = b.colors.size() / 3;
    out->vertices = b.vertices.data();
    out->normals = b.normals.data();
    out->colors = b.colors.data();
    out->triangles = b.triangles.data();
  });
}
vxm_status vxm_mesh_layer_erase(vxm_mesh_layer* m, const vxm_grid_index* g) {
  return guard([&] {
    REQUIRE_ARG(m && g, "null argument");
    if (coord_ok(g->x) && coord_ok(g->y) && coord_ok(g->z)) m->blocks.erase(pack_key(g->x, g->y, g->z));
  });
}
vxm_status vxm_mesh_block(vxm_mesh_layer* m, vxm_layer* T, const vxm_grid_index* g, const vxm_mesh_config* cfg,
                          vxm_layer* color) {
  return guard([&] {
    REQUIRE_ARG(m && T && g && cfg, "null argument");
    REQUIRE_ARG(T->type == VXM_LAYER_TSDF, "mesh_block: source is not a TSDF layer");
    REQUIRE_ARG(!color || color->type == VXM_LAYER_COLOR, "mesh_block: color is not a color layer");
    vxm_blocklist one;
    one.ctx = T->ctx;
    one.assign_host(g, 1);
    T->refresh();
    run_mesh_blocks(m, T, &one, cfg->min_weight, color);
  });
}
vxm_status vxm_update_mesh_list(vxm_mesh_layer* m, vxm_layer* T, vxm_blocklist* updated,
                                const vxm_mesh_config* cfg, vxm_layer* color, vxm_blocklist* out) {
  return guard([&] {
    REQUIRE_ARG(m && T && updated && cfg && out, "null argument");
    REQUIRE_ARG(T->type == VXM_LAYER_TSDF, "update_mesh: source is not a TSDF layer");
    REQUIRE_ARG(!color || color->type == VXM_LAYER_COLOR, "update_mesh: color is not a color layer");
    const auto targets = run_update_mesh(m, T, updated, cfg->min_weight, color);
    out->bind(T->ctx);
    out->assign_host(targets.data(), targets.size());
    out->sorted_unique = true;
  });
}
vxm_status vxm_update_mesh(vxm_mesh_layer* m, vxm_layer* T, const vxm_grid_index* updated, uint64_t n,
                           const vxm_mesh_config* cfg, vxm_layer* color, vxm_blocklist* out) {
  return guard([&] {
    REQUIRE_ARG(T && (updated || n == 0), "null argument");
    vxm_blocklist list;
    list.ctx = T->ctx;
    list.assign_host(updated, n);
    const vxm_status s = vxm_update_mesh_list(m, T, &list, cfg, color, out);
    if (s != VXM_OK) throw Error(s, g_err);
  });
}
vxm_status vxm_save_mesh_ply(const vxm_mesh_layer* m, const char* path) {
  return guard([&] {
    REQUIRE_ARG(m && path, "null argument");
    write_ply(*m, path);
  });
}
}  // extern "C"
