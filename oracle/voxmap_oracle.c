/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (plain-C restatement) of the
 * reference's per-frame map update.  See voxmap_oracle.h for the contract.
 * Every function cites the reference file:line (under /root/reference/proj)
 * whose semantics it restates.  Arithmetic follows the pinned association
 * order of oracle/eigen_shim: 3-term sums are a0 + (a1 + a2).
 */
#define _GNU_SOURCE
#include "voxmap_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* vxo_last_error(void) { return g_err; }
void vxo_free(void* p) { free(p); }

/* ------------------------------------------------------------------------ */
/* Index algebra — include/voxmap/core/indexing.hpp:28-140                   */

#define VPS 8
#define VPB 512

typedef vxm_grid_index gidx;

static int gidx_cmp(const void* a, const void* b) { /* operator<=> indexing.hpp:38 */
  const gidx* x = (const gidx*)a;
  const gidx* y = (const gidx*)b;
  if (x->x != y->x) return x->x < y->x ? -1 : 1;
  if (x->y != y->y) return x->y < y->y ? -1 : 1;
  if (x->z != y->z) return x->z < y->z ? -1 : 1;
  return 0;
}
static int gidx_eq(gidx a, gidx b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

/* floor_div_side — indexing.hpp:71-73 */
static int64_t floor_div_side(int64_t a) {
  return a >= 0 ? a / VPS : -((-a + VPS - 1) / VPS);
}

/* Eigen-shim 3-term sum order. */
static inline double sum3(double a0, double a1, double a2) { return a0 + (a1 + a2); }

/* Pose::operator*(Vector3d) — pose.hpp:58-60: R*p + t, rows a0 + (a1 + a2). */
static inline void pose_apply(const vxm_pose* T, const double p[3], double out[3]) {
  for (int i = 0; i < 3; ++i)
    out[i] = sum3(T->R[3 * i] * p[0], T->R[3 * i + 1] * p[1], T->R[3 * i + 2] * p[2]) + T->t[i];
}

/* Pose::inverse — pose.hpp:52: {R^T, -(R^T t)}. */
void vxo_pose_inverse(const vxm_pose* T, vxm_pose* out) {
  vxm_pose o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.R[3 * r + c] = T->R[3 * c + r];
  for (int i = 0; i < 3; ++i)
    o.t[i] = -sum3(o.R[3 * i] * T->t[0], o.R[3 * i + 1] * T->t[1], o.R[3 * i + 2] * T->t[2]);
  *out = o;
}

/* Pose::valid — pose.hpp:42-50. */
int vxo_pose_valid(const vxm_pose* T) {
  for (int i = 0; i < 9; ++i)
    if (!isfinite(T->R[i])) return 0;
  for (int i = 0; i < 3; ++i)
    if (!isfinite(T->t[i])) return 0;
  const double* m = T->R; /* m[r*3+c] */
#define M(r, c) m[(r) * 3 + (c)]
  /* Eigen bruteforce det3: h(0,1,2) - h(1,0,2) + h(2,0,1), h(a,b,c) = m0a*(m1b*m2c - m1c*m2b) */
  const double h012 = M(0, 0) * (M(1, 1) * M(2, 2) - M(1, 2) * M(2, 1));
  const double h102 = M(0, 1) * (M(1, 0) * M(2, 2) - M(1, 2) * M(2, 0));
  const double h201 = M(0, 2) * (M(1, 0) * M(2, 1) - M(1, 1) * M(2, 0));
  const double det = h012 - h102 + h201;
  double ortho = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      /* (R^T R)(r,c) = sum_k R(k,r) R(k,c) */
      const double v = sum3(M(0, r) * M(0, c), M(1, r) * M(1, c), M(2, r) * M(2, c)) -
                       (r == c ? 1.0 : 0.0);
      const double a = fabs(v);
      ortho = ortho < a ? a : ortho;
    }
#undef M
  return fabs(det - 1.0) <= 1e-6 && ortho <= 1e-6;
}

/* ------------------------------------------------------------------------ */
/* Hash set / map of GridIndex (stands in for std::unordered_map/set)        */

typedef struct {
  gidx* keys;
  int64_t* vals;
  uint8_t* used;
  uint64_t cap, n;
} gmap;

static uint64_t ghash(gidx g) {
  uint64_t h = (uint64_t)(uint32_t)g.x * 0x9E3779B97F4A7C15ull;
  h ^= (uint64_t)(uint32_t)g.y * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
  h ^= (uint64_t)(uint32_t)g.z * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
  return h ^ (h >> 29);
}
static void gmap_init(gmap* m, uint64_t cap) {
  uint64_t c = 16;
  while (c < cap * 2) c <<= 1;
  m->cap = c;
  m->n = 0;
  m->keys = (gidx*)malloc(sizeof(gidx) * c);
  m->vals = (int64_t*)malloc(sizeof(int64_t) * c);
  m->used = (uint8_t*)calloc(c, 1);
}
static void gmap_free(gmap* m) {
  free(m->keys);
  free(m->vals);
  free(m->used);
  memset(m, 0, sizeof *m);
}
static int64_t gmap_get(const gmap* m, gidx g) {
  if (!m->cap) return -1;
  uint64_t i = ghash(g) & (m->cap - 1);
  while (m->used[i]) {
    if (gidx_eq(m->keys[i], g)) return m->vals[i];
    i = (i + 1) & (m->cap - 1);
  }
  return -1;
}
static void gmap_put(gmap* m, gidx g, int64_t v);
static void gmap_grow(gmap* m) {
  gmap n;
  gmap_init(&n, m->cap);
  for (uint64_t i = 0; i < m->cap; ++i)
    if (m->used[i]) gmap_put(&n, m->keys[i], m->vals[i]);
  gmap_free(m);
  *m = n;
}
/* insert-if-absent; returns 1 when inserted */
static int gmap_insert(gmap* m, gidx g, int64_t v) {
  if (!m->cap) gmap_init(m, 64);
  if ((m->n + 1) * 2 > m->cap) gmap_grow(m);
  uint64_t i = ghash(g) & (m->cap - 1);
  while (m->used[i]) {
    if (gidx_eq(m->keys[i], g)) return 0;
    i = (i + 1) & (m->cap - 1);
  }
  m->used[i] = 1;
  m->keys[i] = g;
  m->vals[i] = v;
  m->n++;
  return 1;
}
static void gmap_put(gmap* m, gidx g, int64_t v) { gmap_insert(m, g, v); }

/* growable GridIndex vector */
typedef struct {
  gidx* v;
  uint64_t n, cap;
} gvec;
static void gvec_push(gvec* a, gidx g) {
  if (a->n == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 64;
    a->v = (gidx*)realloc(a->v, sizeof(gidx) * a->cap);
  }
  a->v[a->n++] = g;
}
static void gvec_sort_unique(gvec* a) { /* sort_unique esdf/integrator.cpp:39-42 */
  if (!a->n) return;
  qsort(a->v, a->n, sizeof(gidx), gidx_cmp);
  uint64_t k = 1;
  for (uint64_t i = 1; i < a->n; ++i)
    if (!gidx_eq(a->v[i], a->v[k - 1])) a->v[k++] = a->v[i];
  a->n = k;
}
static void gvec_emit(gvec* a, vxm_grid_index** out, uint64_t* n) {
  *out = a->v ? a->v : (gidx*)malloc(sizeof(gidx));
  *n = a->n;
  a->v = NULL;
  a->n = a->cap = 0;
}

/* ------------------------------------------------------------------------ */
/* Layer<V> — include/voxmap/core/layer.hpp:47-125                          */

struct vxo_layer {
  int type; /* VXM_LAYER_TSDF / VXM_LAYER_ESDF / VXM_LAYER_OCCUPANCY */
  double vs;
  uint64_t max_blocks;
  size_t vbytes; /* voxel bytes */
  gmap index;    /* key -> block number */
  gidx* keys;    /* block number -> key */
  unsigned char* data;
  uint64_t n, cap;
};

int vxo_layer_create(int type, double vs, uint64_t max_blocks, vxo_layer** out) {
  if (!(vs > 0.0)) return fail(VXM_ERR_INVALID_ARGUMENT, "Layer: voxel_size must be positive");
  vxo_layer* L = (vxo_layer*)calloc(1, sizeof *L);
  L->type = type;
  L->vs = vs;
  L->max_blocks = max_blocks ? max_blocks : (1ull << 30);
  L->vbytes = type == VXM_LAYER_TSDF   ? sizeof(vxm_tsdf_voxel)
              : type == VXM_LAYER_ESDF ? sizeof(vxm_esdf_voxel)
                                       : sizeof(vxm_occupancy_voxel);
  *out = L;
  return VXM_OK;
}
void vxo_layer_destroy(vxo_layer* L) {
  if (!L) return;
  gmap_free(&L->index);
  free(L->keys);
  free(L->data);
  free(L);
}
uint64_t vxo_layer_num_blocks(const vxo_layer* L) { return L->n; }
static size_t block_bytes(const vxo_layer* L) { return L->vbytes * VPB; }
static void* block_ptr(const vxo_layer* L, gidx g) { /* layer.hpp:65-72 */
  const int64_t i = gmap_get(&L->index, g);
  return i < 0 ? NULL : L->data + (size_t)i * block_bytes(L);
}
static int has_block(const vxo_layer* L, gidx g) { return gmap_get(&L->index, g) >= 0; }
/* get_or_allocate — layer.hpp:74-86: zero block, MapCapacityError when full. */
static void* get_or_allocate(vxo_layer* L, gidx g, int* err) {
  const int64_t i = gmap_get(&L->index, g);
  if (i >= 0) return L->data + (size_t)i * block_bytes(L);
  if (L->n >= L->max_blocks) {
    *err = fail(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
    return NULL;
  }
  if (L->n == L->cap) {
    L->cap = L->cap ? L->cap * 2 : 256;
    L->data = (unsigned char*)realloc(L->data, L->cap * block_bytes(L));
    L->keys = (gidx*)realloc(L->keys, L->cap * sizeof(gidx));
  }
  memset(L->data + L->n * block_bytes(L), 0, block_bytes(L));
  L->keys[L->n] = g;
  gmap_insert(&L->index, g, (int64_t)L->n);
  return L->data + (L->n++) * block_bytes(L);
}
static gvec sorted_indices(const vxo_layer* L) { /* layer.hpp:109-117 */
  gvec a = {0};
  for (uint64_t i = 0; i < L->n; ++i) gvec_push(&a, L->keys[i]);
  if (a.n) qsort(a.v, a.n, sizeof(gidx), gidx_cmp);
  return a;
}
int vxo_layer_export(const vxo_layer* L, vxm_grid_index* keys, void* voxels) {
  gvec a = sorted_indices(L);
  for (uint64_t i = 0; i < a.n; ++i) {
    keys[i] = a.v[i];
    if (voxels)
      memcpy((char*)voxels + i * block_bytes(L), block_ptr(L, a.v[i]), block_bytes(L));
  }
  free(a.v);
  return VXM_OK;
}
int vxo_layer_write_blocks(vxo_layer* L, const vxm_grid_index* keys, uint64_t n,
                           const void* voxels) {
  for (uint64_t i = 0; i < n; ++i) {
    int err = 0;
    void* b = get_or_allocate(L, keys[i], &err);
    if (!b) return err;
    memcpy(b, (const char*)voxels + i * block_bytes(L), block_bytes(L));
  }
  return VXM_OK;
}

/* ------------------------------------------------------------------------ */
/* Sensors — sensor/camera.hpp, sensor/lidar.hpp, sensor/image.hpp           */

static const double kTwoPi = 2.0 * 3.14159265358979323846;

static inline int valid_depth(float d) { return d > 0.0f && isfinite(d); } /* image.hpp:38 */

/* LidarIntrinsics::ray_direction — lidar.hpp:68-74 */
static void lidar_ray_direction(const vxm_lidar* l, double u, double v, double out[3]) {
  const double az = l->azimuth_start + u * (l->azimuth_fov / l->num_azimuth);
  const double polar = l->elevation_start + v * (l->elevation_fov / l->num_elevation);
  const double sp = sin(polar);
  out[0] = cos(az) * sp;
  out[1] = sin(az) * sp;
  out[2] = cos(polar);
}
/* p.norm() with the shim order: sqrt(x^2 + (y^2 + z^2)) */
static inline double norm3(const double p[3]) {
  return sqrt(sum3(p[0] * p[0], p[1] * p[1], p[2] * p[2]));
}
/* LidarIntrinsics::project — lidar.hpp:43-55 (includes contains()). */
static int lidar_project(const vxm_lidar* l, const double p[3], double* u, double* v) {
  const double r = norm3(p);
  if (!(r > 0.0)) return 0;
  double az = atan2(p[1], p[0]) - l->azimuth_start;
  az -= kTwoPi * floor(az / kTwoPi);
  *u = az * (l->num_azimuth / l->azimuth_fov);
  double c = p[2] / r;
  c = c < -1.0 ? -1.0 : (1.0 < c ? 1.0 : c); /* std::clamp */
  const double polar = acos(c);
  *v = (polar - l->elevation_start) * (l->num_elevation / l->elevation_fov);
  return *u >= 0.0 && *u < l->num_azimuth && *v >= 0.0 && *v < l->num_elevation;
}

/* sample_depth_nearest — image.hpp:65-74 */
static int sample_nearest(const float* img, int W, int H, double u, double v, float* out) {
  const int col = (int)floor(u);
  const int row = (int)floor(v);
  if (u < 0.0 || v < 0.0 || col >= W || row >= H) return 0;
  const float d = img[(size_t)row * W + col];
  if (!valid_depth(d)) return 0;
  *out = d;
  return 1;
}
/* sample_depth_linear — image.hpp:79-106 */
static int sample_linear(const float* img, int W, int H, double u, double v, float gap,
                         float* out) {
  const double gu = u - 0.5, gv = v - 0.5;
  const int x0 = (int)floor(gu), y0 = (int)floor(gv);
  if (x0 < 0 || y0 < 0 || x0 + 1 >= W || y0 + 1 >= H) return 0;
  const float d00 = img[(size_t)y0 * W + x0], d10 = img[(size_t)y0 * W + x0 + 1];
  const float d01 = img[(size_t)(y0 + 1) * W + x0], d11 = img[(size_t)(y0 + 1) * W + x0 + 1];
  if (!valid_depth(d00) || !valid_depth(d10) || !valid_depth(d01) || !valid_depth(d11)) return 0;
  float lo = d00, hi = d00;
  const float c[3] = {d10, d01, d11};
  for (int i = 0; i < 3; ++i) {
    lo = c[i] < lo ? c[i] : lo;
    hi = hi < c[i] ? c[i] : hi;
  }
  if (hi - lo > gap) return 0;
  const double wx = gu - x0, wy = gv - y0;
  const double d = (1.0 - wy) * ((1.0 - wx) * d00 + wx * d10) + wy * ((1.0 - wx) * d01 + wx * d11);
  *out = (float)d;
  return 1;
}

/* ------------------------------------------------------------------------ */
/* View candidates — sensor/traversal.hpp:29-73, sensor/view.cpp:25-111      */

/* traverse_grid — traversal.hpp:29-73 */
static void traverse_grid(const double s[3], const double e[3], double cs, gmap* touched) {
  double d[3];
  int cell[3], end_cell[3], step[3] = {0, 0, 0};
  double t_max[3] = {INFINITY, INFINITY, INFINITY}, t_delta[3] = {INFINITY, INFINITY, INFINITY};
  for (int i = 0; i < 3; ++i) {
    d[i] = e[i] - s[i];
    cell[i] = (int)floor(s[i] / cs);
    end_cell[i] = (int)floor(e[i] / cs);
  }
  for (int i = 0; i < 3; ++i) {
    if (d[i] > 0.0) {
      step[i] = 1;
      t_delta[i] = cs / d[i];
      t_max[i] = ((cell[i] + 1) * cs - s[i]) / d[i];
    } else if (d[i] < 0.0) {
      step[i] = -1;
      t_delta[i] = -cs / d[i];
      t_max[i] = (cell[i] * cs - s[i]) / d[i];
    }
  }
  gidx g = {cell[0], cell[1], cell[2]};
  gmap_insert(touched, g, 0);
  int guard = abs(end_cell[0] - cell[0]) + abs(end_cell[1] - cell[1]) + abs(end_cell[2] - cell[2]) + 3;
  while (guard-- > 0) {
    int axis = 0;
    if (t_max[1] < t_max[0]) axis = 1;
    if (t_max[2] < t_max[axis]) axis = 2;
    if (t_max[axis] > 1.0) break;
    cell[axis] += step[axis];
    t_max[axis] += t_delta[axis];
    gidx h = {cell[0], cell[1], cell[2]};
    gmap_insert(touched, h, 0);
  }
}

/* dilate_and_sort — view.cpp:25-41 */
static gvec dilate_and_sort(const gmap* touched) {
  gmap out = {0};
  gmap_init(&out, touched->n * 27 + 16);
  gvec res = {0};
  for (uint64_t i = 0; i < touched->cap; ++i) {
    if (!touched->used[i]) continue;
    const gidx g = touched->keys[i];
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          gidx h = {g.x + dx, g.y + dy, g.z + dz};
          if (gmap_insert(&out, h, 0)) gvec_push(&res, h);
        }
  }
  gmap_free(&out);
  if (res.n) qsort(res.v, res.n, sizeof(gidx), gidx_cmp);
  return res;
}

/* cast_ray — view.cpp:45-57 (end_S supplied by the sensor-specific caller) */
static void cast_ray_end(const vxm_pose* T, const double end_S[3], double cs, gmap* touched) {
  double end_L[3];
  pose_apply(T, end_S, end_L);
  traverse_grid(T->t, end_L, cs, touched);
}
static double ray_reach(double depth, const vxm_view_config* cfg) {
  const double capped = cfg->max_integration_distance < depth ? cfg->max_integration_distance : depth;
  return capped + cfg->truncation;
}

static gvec view_camera(const vxm_pose* T, const vxm_camera* cam, const float* depth, int W, int H,
                        double cs, const vxm_view_config* cfg) { /* view.cpp:61-92 */
  gmap touched = {0};
  gmap_init(&touched, 4096);
  const int tile = cfg->pixel_subsample > 1 ? cfg->pixel_subsample : 1;
  for (int row0 = 0; row0 < H; row0 += tile) {
    for (int col0 = 0; col0 < W; col0 += tile) {
      float tile_max = 0.0f;
      const int row1 = row0 + tile < H ? row0 + tile : H;
      const int col1 = col0 + tile < W ? col0 + tile : W;
      for (int r = row0; r < row1; ++r)
        for (int c = col0; c < col1; ++c) {
          const float d = depth[(size_t)r * W + c];
          if (valid_depth(d)) tile_max = tile_max < d ? d : tile_max;
        }
      if (tile_max <= 0.0f) continue;
      const double u = 0.5 * (col0 + col1), v = 0.5 * (row0 + row1);
      const double reach = ray_reach((double)tile_max, cfg);
      /* CameraIntrinsics::unproject — camera.hpp:52-55 */
      const double end_S[3] = {(u - cam->cu) / cam->fu * reach, (v - cam->cv) / cam->fv * reach,
                               reach};
      cast_ray_end(T, end_S, cs, &touched);
    }
  }
  gvec out = dilate_and_sort(&touched);
  gmap_free(&touched);
  return out;
}

static gvec view_lidar(const vxm_pose* T, const vxm_lidar* li, const float* depth, int W, int H,
                       double cs, const vxm_view_config* cfg) { /* view.cpp:94-111 */
  gmap touched = {0};
  gmap_init(&touched, 1 << 16);
  for (int row = 0; row < H; ++row)
    for (int col = 0; col < W; ++col) {
      const float d = depth[(size_t)row * W + col];
      if (!valid_depth(d)) continue;
      const double reach = ray_reach((double)d, cfg);
      double dir[3];
      lidar_ray_direction(li, col + 0.5, row + 0.5, dir); /* unproject lidar.hpp:64-66 */
      const double end_S[3] = {dir[0] * reach, dir[1] * reach, dir[2] * reach};
      cast_ray_end(T, end_S, cs, &touched);
    }
  gvec out = dilate_and_sort(&touched);
  gmap_free(&touched);
  return out;
}

int vxo_blocks_in_view_camera(const vxm_pose* T, const vxm_camera* cam, const float* depth, int w,
                              int h, double cs, const vxm_view_config* cfg, vxm_grid_index** out,
                              uint64_t* n) {
  gvec a = view_camera(T, cam, depth, w, h, cs, cfg);
  gvec_emit(&a, out, n);
  return VXM_OK;
}
int vxo_blocks_in_view_lidar(const vxm_pose* T, const vxm_lidar* li, const float* depth, int w,
                             int h, double cs, const vxm_view_config* cfg, vxm_grid_index** out,
                             uint64_t* n) {
  gvec a = view_lidar(T, li, depth, w, h, cs, cfg);
  gvec_emit(&a, out, n);
  return VXM_OK;
}

/* ------------------------------------------------------------------------ */
/* TSDF integration — integrate/integrator.cpp:26-146, updates.hpp:27-54     */

/* tsdf_update — updates.hpp:39-54 (std::clamp / std::min forms) */
static vxm_tsdf_voxel tsdf_update(vxm_tsdf_voxel vox, float d_p, float w_new,
                                  const vxm_integrator_config* cfg) {
  const float eps = (float)cfg->truncation;
  if (d_p < -eps) return vox;
  const float d_t = d_p < -eps ? -eps : (eps < d_p ? eps : d_p);
  vxm_tsdf_voxel out;
  const float w_sum = vox.weight + w_new;
  const float avg = (vox.weight * vox.distance + w_new * d_t) / w_sum;
  out.distance = avg < -eps ? -eps : (eps < avg ? eps : avg);
  out.weight = cfg->max_weight < w_sum ? cfg->max_weight : w_sum;
  return out;
}
/* quantize_log_odds — integrate/config.hpp:29-31 */
static float quantize_log_odds(float v) { return (float)(nearbyint((double)v * 4096.0) / 4096.0); }
/* occupancy_update — updates.hpp:59-72 */
static float occupancy_update(float lo, float d_p, const vxm_integrator_config* cfg) {
  const float eps = (float)cfg->truncation;
  if (d_p < -eps) return lo;
  const float inc = d_p <= 0.0f ? quantize_log_odds(cfg->hit_log_odds)
                                : quantize_log_odds(cfg->miss_log_odds);
  const float v = lo + inc;
  const float lo_min = quantize_log_odds(cfg->log_odds_min), lo_max = quantize_log_odds(cfg->log_odds_max);
  return v < lo_min ? lo_min : (lo_max < v ? lo_max : v);
}
/* weight_for_depth — updates.hpp:27-32 */
static float weight_for_depth(double d, const vxm_integrator_config* cfg) {
  if (cfg->weighting == VXM_WEIGHT_INVERSE_SQUARE) {
    const double dd = d * d;
    return (float)(1.0 / (dd < 1e-6 ? 1e-6 : dd));
  }
  return 1.0f;
}

static int check_frame(const vxm_pose* T, int iw, int ih, int sw, int sh) { /* integrator.cpp:26-34 */
  if (!vxo_pose_valid(T)) return fail(VXM_ERR_INVALID_POSE, "integrate: degenerate sensor pose");
  if (iw != sw || ih != sh)
    return fail(VXM_ERR_INVALID_ARGUMENT, "integrate: image size does not match intrinsics");
  return VXM_OK;
}

/* integrate_impl — integrator.cpp:71-134 */
static int integrate_impl(vxo_layer* L, const float* depth, int W, int H, const vxm_pose* T,
                          const vxm_camera* cam, const vxm_lidar* li,
                          const vxm_integrator_config* cfg, vxm_grid_index** out, uint64_t* n) {
  int rc = cam ? check_frame(T, W, H, cam->width, cam->height)
               : check_frame(T, W, H, li->num_azimuth, li->num_elevation);
  if (rc) return rc;
  const vxm_view_config vc = {cfg->max_integration_distance, cfg->truncation,
                              cfg->view_pixel_subsample};
  const double cs = L->vs * VPS;
  gvec cand = cam ? view_camera(T, cam, depth, W, H, cs, &vc) : view_lidar(T, li, depth, W, H, cs, &vc);
  /* allocation loop — integrator.cpp:84-87 (serial, sorted order) */
  for (uint64_t i = 0; i < cand.n; ++i) {
    int err = 0;
    if (!get_or_allocate(L, cand.v[i], &err)) {
      free(cand.v);
      return err;
    }
  }
  vxm_pose Tsl;
  vxo_pose_inverse(T, &Tsl);
  const int mode = cam ? cfg->camera_sample : cfg->lidar_sample;
  const double vs = L->vs;
  const double max_voxel_depth = cfg->max_integration_distance + cfg->truncation;
  gvec changed = {0};
  for (uint64_t i = 0; i < cand.n; ++i) {
    const gidx g = cand.v[i];
    vxm_tsdf_voxel* blk = (vxm_tsdf_voxel*)block_ptr(L, g);
    float* oblk = (float*)blk; /* Layer<OccupancyVoxel> (integrator.cpp:148-158) */
    const int occ = L->type == VXM_LAYER_OCCUPANCY;
    int block_changed = 0;
    for (int lin = 0; lin < VPB; ++lin) {
      const int vx = lin % VPS, vy = (lin / VPS) % VPS, vz = lin / (VPS * VPS);
      /* voxel_center — indexing.hpp:113-119 */
      const double c[3] = {((double)g.x * VPS + vx + 0.5) * vs, ((double)g.y * VPS + vy + 0.5) * vs,
                           ((double)g.z * VPS + vz + 0.5) * vs};
      double p[3];
      pose_apply(&Tsl, c, p);
      const double d_v = cam ? p[2] : norm3(p);
      if (!(d_v > 0.0) || d_v > max_voxel_depth) continue;
      double u = 0.0, w = 0.0;
      if (cam) { /* CameraIntrinsics::project + contains — camera.hpp:35-46 */
        if (!(p[2] > 0.0)) continue;
        u = cam->fu * p[0] / p[2] + cam->cu;
        w = cam->fv * p[1] / p[2] + cam->cv;
        if (!(u >= 0.0 && u < cam->width && w >= 0.0 && w < cam->height)) continue;
      } else {
        if (!lidar_project(li, p, &u, &w)) continue;
      }
      float s;
      const int ok = mode == VXM_SAMPLE_NEAREST ? sample_nearest(depth, W, H, u, w, &s)
                                                : sample_linear(depth, W, H, u, w, cfg->max_sample_gap, &s);
      if (!ok) continue;
      const float d_p = s - (float)d_v;
      if (occ) {
        const float nv = occupancy_update(oblk[lin], d_p, cfg);
        if (memcmp(&nv, &oblk[lin], sizeof nv) != 0) {
          oblk[lin] = nv;
          block_changed = 1;
        }
        continue;
      }
      const vxm_tsdf_voxel nv = tsdf_update(blk[lin], d_p, weight_for_depth((double)s, cfg), cfg);
      if (memcmp(&nv, &blk[lin], sizeof nv) != 0) {
        blk[lin] = nv;
        block_changed = 1;
      }
    }
    if (block_changed) gvec_push(&changed, g);
  }
  free(cand.v);
  gvec_emit(&changed, out, n);
  return VXM_OK;
}

int vxo_integrate_camera(vxo_layer* L, const float* depth, int w, int h, const vxm_pose* T,
                         const vxm_camera* cam, const vxm_integrator_config* cfg,
                         vxm_grid_index** out, uint64_t* n) {
  return integrate_impl(L, depth, w, h, T, cam, NULL, cfg, out, n);
}
int vxo_integrate_lidar(vxo_layer* L, const float* depth, int w, int h, const vxm_pose* T,
                        const vxm_lidar* li, const vxm_integrator_config* cfg, vxm_grid_index** out,
                        uint64_t* n) {
  return integrate_impl(L, depth, w, h, T, NULL, li, cfg, out, n);
}

/* ------------------------------------------------------------------------ */
/* ESDF — esdf/integrator.hpp:26-120, src/esdf/integrator.cpp:26-572         */

typedef vxm_esdf_voxel ev_t;

typedef struct {
  int32_t max_sq, cap_sq;
} limits_t;

static limits_t limits_for(const vxm_esdf_config* cfg, double vs) { /* esdf/integrator.hpp:43-54 */
  const double r = cfg->max_distance / vs;
  limits_t l;
  l.max_sq = (int32_t)llround(r * r);
  l.cap_sq = l.max_sq < 16 ? l.max_sq : 16;
  return l;
}
static inline int ev_observed(const ev_t* v) { return v->flags & VXM_ESDF_OBSERVED; }
static inline int ev_site(const ev_t* v) { return v->flags & VXM_ESDF_SITE; }
static inline int ev_inside(const ev_t* v) { return v->flags & VXM_ESDF_INSIDE; }
static inline int ev_has_parent(const ev_t* v) {
  return v->parent_x != 0 || v->parent_y != 0 || v->parent_z != 0;
}
static inline int ev_eq(const ev_t* a, const ev_t* b) {
  return a->squared_distance == b->squared_distance && a->parent_x == b->parent_x &&
         a->parent_y == b->parent_y && a->parent_z == b->parent_z && a->flags == b->flags &&
         a->reserved == b->reserved;
}
static void reset_to_saturated(ev_t* v, limits_t lim) { /* esdf/integrator.cpp:46-51 */
  v->squared_distance = ev_inside(v) ? lim.cap_sq : lim.max_sq;
  v->parent_x = v->parent_y = v->parent_z = 0;
}

/* relax — esdf/integrator.cpp:58-88 */
static int relax(ev_t* v, const ev_t* u, int dx, int dy, int dz, limits_t lim) {
  if (!ev_observed(u) || (!ev_site(u) && !ev_has_parent(u))) return 0;
  if (!ev_observed(v) || ev_site(v)) return 0;
  const int cx = u->parent_x - dx, cy = u->parent_y - dy, cz = u->parent_z - dz;
  const int32_t cand = (int32_t)((uint32_t)(cx * cx) + (uint32_t)(cy * cy) + (uint32_t)(cz * cz));
  if (cand == 0) return 0;
  const int32_t limit = ev_inside(v) ? lim.cap_sq : lim.max_sq;
  if (cand > limit || cand > v->squared_distance) return 0;
  if (cand == v->squared_distance && ev_has_parent(v)) {
    const int vx = v->parent_x, vy = v->parent_y, vz = v->parent_z;
    const int less = cx < vx || (cx == vx && (cy < vy || (cy == vy && cz < vz)));
    if (!less) return 0;
  }
  v->squared_distance = cand;
  v->parent_x = (int16_t)cx;
  v->parent_y = (int16_t)cy;
  v->parent_z = (int16_t)cz;
  return 1;
}

static inline int lin_of(int x, int y, int z) { return x + VPS * (y + VPS * z); }

/* sweep_block — esdf/integrator.cpp:96-139 */
static int sweep_block(ev_t* b, limits_t lim) {
  int block_changed = 0, pass_changed = 1;
  while (pass_changed) {
    pass_changed = 0;
    for (int z = 0; z < VPS; ++z)
      for (int y = 0; y < VPS; ++y) {
        ev_t* row = b + lin_of(0, y, z);
        for (int x = 1; x < VPS; ++x) pass_changed |= relax(&row[x], &row[x - 1], 1, 0, 0, lim);
        for (int x = VPS - 2; x >= 0; --x) pass_changed |= relax(&row[x], &row[x + 1], -1, 0, 0, lim);
      }
    for (int z = 0; z < VPS; ++z)
      for (int x = 0; x < VPS; ++x) {
        ev_t* col = b + lin_of(x, 0, z);
        for (int y = 1; y < VPS; ++y)
          pass_changed |= relax(&col[y * VPS], &col[(y - 1) * VPS], 0, 1, 0, lim);
        for (int y = VPS - 2; y >= 0; --y)
          pass_changed |= relax(&col[y * VPS], &col[(y + 1) * VPS], 0, -1, 0, lim);
      }
    for (int y = 0; y < VPS; ++y)
      for (int x = 0; x < VPS; ++x) {
        ev_t* pil = b + lin_of(x, y, 0);
        for (int z = 1; z < VPS; ++z)
          pass_changed |= relax(&pil[z * 64], &pil[(z - 1) * 64], 0, 0, 1, lim);
        for (int z = VPS - 2; z >= 0; --z)
          pass_changed |= relax(&pil[z * 64], &pil[(z + 1) * 64], 0, 0, -1, lim);
      }
    block_changed |= pass_changed;
  }
  return block_changed;
}

/* exchange_pair — esdf/integrator.cpp:144-168 */
static void exchange_pair(ev_t* a, ev_t* b, int axis, limits_t lim, int* ac, int* bc) {
  const int dx = axis == 0, dy = axis == 1, dz = axis == 2;
  for (int j = 0; j < VPS; ++j)
    for (int i = 0; i < VPS; ++i) {
      int ax, ay, az, bx, by, bz;
      if (axis == 0) { ax = VPS - 1; ay = i; az = j; bx = 0; by = i; bz = j; }
      else if (axis == 1) { ax = i; ay = VPS - 1; az = j; bx = i; by = 0; bz = j; }
      else { ax = i; ay = j; az = VPS - 1; bx = i; by = j; bz = 0; }
      ev_t* va = a + lin_of(ax, ay, az);
      ev_t* vb = b + lin_of(bx, by, bz);
      *bc |= relax(vb, va, dx, dy, dz, lim);
      *ac |= relax(va, vb, -dx, -dy, -dz, lim);
    }
}

struct vxo_state { /* EsdfUpdateState — esdf/integrator.hpp:67-74 */
  gvec lists[3]; /* to_update, to_clear, cleared */
};
vxo_state* vxo_state_create(void) { return (vxo_state*)calloc(1, sizeof(vxo_state)); }
void vxo_state_destroy(vxo_state* s) {
  if (!s) return;
  for (int i = 0; i < 3; ++i) free(s->lists[i].v);
  free(s);
}
int vxo_state_get(vxo_state* s, int which, vxm_grid_index** out, uint64_t* n) {
  gvec c = {0};
  for (uint64_t i = 0; i < s->lists[which].n; ++i) gvec_push(&c, s->lists[which].v[i]);
  gvec_emit(&c, out, n);
  return VXM_OK;
}
int vxo_state_set(vxo_state* s, int which, const vxm_grid_index* k, uint64_t n) {
  s->lists[which].n = 0;
  for (uint64_t i = 0; i < n; ++i) gvec_push(&s->lists[which], k[i]);
  return VXM_OK;
}

static gidx gstep(gidx g, int axis, int s) {
  if (axis == 0) g.x += s;
  else if (axis == 1) g.y += s;
  else g.z += s;
  return g;
}

/* OccupancyClassifier — esdf/integrator.cpp:200-266 */
static int occ_observed(float lo) { return lo != 0.0f; }
static int occ_free(float lo, float thr) { return occ_observed(lo) && !(lo > thr); }
static void occ_classify(const vxo_layer* occ, gidx g, const float* blk, int lin, float thr,
                         int* observed, int* site, int* inside) {
  const float lo = blk[lin];
  *observed = occ_observed(lo);
  *site = *inside = 0;
  if (!*observed) return;
  *inside = lo > thr;
  if (!*inside) return; /* free voxels are never sites */
  const int v[3] = {lin % VPS, (lin / VPS) % VPS, lin / (VPS * VPS)};
  for (int n = 0; n < 6; ++n) { /* steps {+x,-x,+y,-y,+z,-z} */
    const int axis = n / 2, step = (n & 1) ? -1 : 1;
    int c[3] = {v[0], v[1], v[2]};
    c[axis] += step;
    const float* nb = NULL;
    if (c[axis] >= 0 && c[axis] < VPS) {
      nb = blk;
    } else {
      nb = (const float*)block_ptr(occ, gstep(g, axis, step));
      c[axis] = (c[axis] + VPS) % VPS;
    }
    if (nb && occ_free(nb[c[0] + VPS * (c[1] + VPS * c[2])], thr)) {
      *site = 1;
      return;
    }
  }
}

/* mark_impl with TsdfClassifier / OccupancyClassifier — esdf/integrator.cpp:177-348 */
static int mark_sites(vxo_layer* esdf, const vxo_layer* tsdf, const gidx* upd, uint64_t nu,
                      const vxm_esdf_config* cfg, vxo_state* st, gvec* changed) {
  const limits_t lim = limits_for(cfg, esdf->vs);
  const float site_threshold = (float)cfg->site_threshold;
  gvec eff = {0};
  for (uint64_t i = 0; i < nu; ++i) {
    const gidx g = upd[i];
    const gidx c7[7] = {g, gstep(g, 0, 1), gstep(g, 0, -1), gstep(g, 1, 1),
                        gstep(g, 1, -1), gstep(g, 2, 1), gstep(g, 2, -1)};
    for (int k = 0; k < 7; ++k)
      if (has_block(tsdf, c7[k])) gvec_push(&eff, c7[k]);
  }
  gvec_sort_unique(&eff);
  for (uint64_t e = 0; e < eff.n; ++e) {
    const gidx g = eff.v[e];
    int err = 0;
    ev_t* blk = (ev_t*)get_or_allocate(esdf, g, &err);
    if (!blk) {
      free(eff.v);
      return err;
    }
    const vxm_tsdf_voxel* src = (const vxm_tsdf_voxel*)block_ptr(tsdf, g);
    int bchanged = 0, bupdate = 0, bclear = 0;
    for (int lin = 0; lin < VPB; ++lin) {
      int observed, site, inside;
      if (tsdf->type == VXM_LAYER_OCCUPANCY) {
        occ_classify(tsdf, g, (const float*)src, lin, cfg->occupied_log_odds_threshold, &observed,
                     &site, &inside);
      } else {
        const vxm_tsdf_voxel tv = src[lin];
        observed = tv.weight > 0.0f;
        site = observed && fabsf(tv.distance) <= site_threshold;
        inside = observed && tv.distance < 0.0f;
      }
      ev_t* ev = &blk[lin];
      ev_t nv = *ev;
      if (!observed) {
        if (ev_site(ev)) bclear = 1;
        memset(&nv, 0, sizeof nv);
      } else {
        nv.flags = (uint8_t)(VXM_ESDF_OBSERVED | (site ? VXM_ESDF_SITE : 0) |
                             (inside ? VXM_ESDF_INSIDE : 0));
        if (site) {
          nv.squared_distance = 0;
          nv.parent_x = nv.parent_y = nv.parent_z = 0;
          if (!ev_observed(ev) || !ev_site(ev)) bupdate = 1;
        } else if (!ev_observed(ev)) {
          reset_to_saturated(&nv, lim);
          bupdate = 1;
        } else if (ev_site(ev)) {
          reset_to_saturated(&nv, lim);
          bclear = 1;
          bupdate = 1;
        } else if (!!ev_inside(ev) != inside) {
          reset_to_saturated(&nv, lim);
          bupdate = 1;
        }
      }
      if (!ev_eq(&nv, ev)) {
        *ev = nv;
        bchanged = 1;
      }
    }
    if (bchanged) gvec_push(changed, g);
    if (bupdate) gvec_push(&st->lists[0], g);
    if (bclear) gvec_push(&st->lists[1], g);
  }
  free(eff.v);
  gvec_sort_unique(&st->lists[0]);
  gvec_sort_unique(&st->lists[1]);
  return VXM_OK;
}

/* clear_invalid — esdf/integrator.cpp:433-486 */
static void clear_invalid(vxo_layer* esdf, const vxm_esdf_config* cfg, vxo_state* st,
                          gvec* changed) {
  if (!st->lists[1].n) return;
  const limits_t lim = limits_for(cfg, esdf->vs);
  const int radius = (int)ceil(cfg->max_distance / esdf->vs / VPS);
  gvec all = sorted_indices(esdf);
  gvec scan = {0};
  for (uint64_t i = 0; i < all.n; ++i) {
    const gidx g = all.v[i];
    for (uint64_t k = 0; k < st->lists[1].n; ++k) {
      const gidx c = st->lists[1].v[k];
      if (abs(g.x - c.x) <= radius && abs(g.y - c.y) <= radius && abs(g.z - c.z) <= radius) {
        gvec_push(&scan, g);
        break;
      }
    }
  }
  /* The reference runs the scanned blocks in parallel; resets only clear
   * parented voxels while reads only test is_site(), so any order gives the
   * same result. */
  for (uint64_t i = 0; i < scan.n; ++i) {
    const gidx g = scan.v[i];
    ev_t* blk = (ev_t*)block_ptr(esdf, g);
    int any = 0;
    for (int lin = 0; lin < VPB; ++lin) {
      ev_t* ev = &blk[lin];
      if (!ev_has_parent(ev)) continue;
      const int vx = lin % VPS, vy = (lin / VPS) % VPS, vz = lin / 64;
      const int64_t px = (int64_t)g.x * VPS + vx + ev->parent_x;
      const int64_t py = (int64_t)g.y * VPS + vy + ev->parent_y;
      const int64_t pz = (int64_t)g.z * VPS + vz + ev->parent_z;
      const gidx pb = {(int32_t)floor_div_side(px), (int32_t)floor_div_side(py),
                       (int32_t)floor_div_side(pz)};
      const ev_t* pblk = (const ev_t*)block_ptr(esdf, pb);
      const ev_t* pv = pblk ? &pblk[lin_of((int)(px - (int64_t)pb.x * VPS),
                                           (int)(py - (int64_t)pb.y * VPS),
                                           (int)(pz - (int64_t)pb.z * VPS))]
                            : NULL;
      if (!pv || !ev_site(pv)) {
        reset_to_saturated(ev, lim);
        any = 1;
      }
    }
    if (any) {
      gvec_push(&st->lists[2], g);
      gvec_push(changed, g);
    }
  }
  free(all.v);
  free(scan.v);
  gvec_sort_unique(&st->lists[2]);
}

/* lower_esdf — esdf/integrator.cpp:488-565 */
static int lower_esdf(vxo_layer* esdf, const gvec* seeds_update, const gvec* seeds_cleared,
                      const vxm_esdf_config* cfg, gvec* changed) {
  const limits_t lim = limits_for(cfg, esdf->vs);
  gvec dirty = {0};
  const gvec* seeds[2] = {seeds_update, seeds_cleared};
  for (int s = 0; s < 2; ++s)
    for (uint64_t i = 0; i < seeds[s]->n; ++i)
      if (has_block(esdf, seeds[s]->v[i])) gvec_push(&dirty, seeds[s]->v[i]);
  gvec_sort_unique(&dirty);
  int rounds = 0;
  gvec changed_set = {0};
  while (dirty.n) {
    ++rounds;
    for (uint64_t i = 0; i < dirty.n; ++i)
      if (sweep_block((ev_t*)block_ptr(esdf, dirty.v[i]), lim)) gvec_push(&changed_set, dirty.v[i]);
    gvec next = {0};
    for (int axis = 0; axis < 3; ++axis) {
      gvec lowers = {0};
      for (uint64_t i = 0; i < dirty.n; ++i) {
        const gidx b = dirty.v[i];
        if (has_block(esdf, gstep(b, axis, 1))) gvec_push(&lowers, b);
        const gidx below = gstep(b, axis, -1);
        if (has_block(esdf, below)) gvec_push(&lowers, below);
      }
      gvec_sort_unique(&lowers);
      for (uint64_t i = 0; i < lowers.n; ++i) {
        const gidx lo = lowers.v[i], hi = gstep(lowers.v[i], axis, 1);
        int ac = 0, bc = 0;
        exchange_pair((ev_t*)block_ptr(esdf, lo), (ev_t*)block_ptr(esdf, hi), axis, lim, &ac, &bc);
        if (ac) {
          gvec_push(&next, lo);
          gvec_push(&changed_set, lo);
        }
        if (bc) {
          gvec_push(&next, hi);
          gvec_push(&changed_set, hi);
        }
      }
      free(lowers.v);
    }
    gvec_sort_unique(&next);
    free(dirty.v);
    dirty = next;
  }
  free(dirty.v);
  gvec_sort_unique(&changed_set);
  for (uint64_t i = 0; i < changed_set.n; ++i) gvec_push(changed, changed_set.v[i]);
  free(changed_set.v);
  return rounds;
}

int vxo_mark_sites(vxo_layer* esdf, const vxo_layer* tsdf, const vxm_grid_index* upd, uint64_t nu,
                   const vxm_esdf_config* cfg, vxo_state* s, vxm_grid_index** out, uint64_t* n) {
  gvec changed = {0};
  const int rc = mark_sites(esdf, tsdf, upd, nu, cfg, s, &changed);
  gvec_emit(&changed, out, n);
  return rc;
}
int vxo_clear_invalid(vxo_layer* esdf, const vxm_esdf_config* cfg, vxo_state* s,
                      vxm_grid_index** out, uint64_t* n) {
  gvec changed = {0};
  clear_invalid(esdf, cfg, s, &changed);
  gvec_emit(&changed, out, n);
  return VXM_OK;
}
int vxo_lower_esdf(vxo_layer* esdf, vxo_state* s, const vxm_esdf_config* cfg, int* rounds,
                   vxm_grid_index** out, uint64_t* n) {
  gvec changed = {0};
  *rounds = lower_esdf(esdf, &s->lists[0], &s->lists[2], cfg, &changed);
  gvec_emit(&changed, out, n);
  return VXM_OK;
}

/* update_impl — esdf/integrator.cpp:365-413 */
int vxo_update_esdf(vxo_layer* esdf, const vxo_layer* tsdf, const vxm_grid_index* upd, uint64_t nu,
                    const vxm_esdf_config* cfg, vxm_grid_index** out, uint64_t* n) {
  gvec changed = {0};
  if (nu == 0) {
    gvec_emit(&changed, out, n);
    return VXM_OK;
  }
  if (esdf->vs != tsdf->vs)
    return fail(VXM_ERR_INVALID_ARGUMENT, "update_esdf: source and ESDF layer voxel sizes differ");
  /* snapshot */
  const uint64_t n_before = esdf->n;
  unsigned char* before = (unsigned char*)malloc(n_before * block_bytes(esdf) + 1);
  memcpy(before, esdf->data, n_before * block_bytes(esdf));
  gmap before_index = {0};
  gmap_init(&before_index, n_before + 16);
  for (uint64_t i = 0; i < n_before; ++i) gmap_insert(&before_index, esdf->keys[i], (int64_t)i);

  vxo_state* st = vxo_state_create();
  gvec touched = {0};
  int rc = mark_sites(esdf, tsdf, upd, nu, cfg, st, &touched);
  if (rc) {
    vxo_state_destroy(st);
    free(touched.v);
    free(before);
    gmap_free(&before_index);
    return rc;
  }
  clear_invalid(esdf, cfg, st, &touched);
  if (st->lists[0].n || st->lists[1].n || st->lists[2].n) {
    /* reset_parented — esdf/integrator.cpp:352-363 */
    const limits_t lim = limits_for(cfg, esdf->vs);
    for (uint64_t b = 0; b < esdf->n; ++b) {
      ev_t* blk = (ev_t*)(esdf->data + b * block_bytes(esdf));
      for (int lin = 0; lin < VPB; ++lin)
        if (ev_observed(&blk[lin]) && !ev_site(&blk[lin]) && ev_has_parent(&blk[lin]))
          reset_to_saturated(&blk[lin], lim);
    }
    gvec all = sorted_indices(esdf);
    gvec none = {0};
    lower_esdf(esdf, &all, &none, cfg, &touched);
    free(all.v);
  }
  gvec all = sorted_indices(esdf);
  for (uint64_t i = 0; i < all.n; ++i) {
    const int64_t bi = gmap_get(&before_index, all.v[i]);
    if (bi < 0 || memcmp(before + (size_t)bi * block_bytes(esdf), block_ptr(esdf, all.v[i]),
                         block_bytes(esdf)) != 0)
      gvec_push(&changed, all.v[i]);
  }
  free(all.v);
  free(touched.v);
  free(before);
  gmap_free(&before_index);
  vxo_state_destroy(st);
  gvec_emit(&changed, out, n);
  return VXM_OK;
}

/* ------------------------------------------------------------------------ */
/* Queries — query/query.cpp:35-161 (production evaluation order)            */

static const ev_t* esdf_voxel_at(const vxo_layer* E, int64_t gx, int64_t gy, int64_t gz) {
  const gidx b = {(int32_t)floor_div_side(gx), (int32_t)floor_div_side(gy),
                  (int32_t)floor_div_side(gz)};
  const ev_t* blk = (const ev_t*)block_ptr(E, b);
  if (!blk) return NULL;
  return &blk[lin_of((int)(gx - (int64_t)b.x * VPS), (int)(gy - (int64_t)b.y * VPS),
                     (int)(gz - (int64_t)b.z * VPS))];
}
static double esdf_distance(const ev_t* v, double vs) { /* esdf/integrator.hpp:59-63 */
  const double d = sqrt((double)v->squared_distance) * vs;
  return ev_inside(v) ? -d : d;
}
static void parent_gradient(const ev_t* v, double g[3]) { /* query.cpp:58-64 */
  g[0] = g[1] = g[2] = 0.0;
  if (!ev_has_parent(v)) return;
  const double off[3] = {(double)v->parent_x, (double)v->parent_y, (double)v->parent_z};
  const double z = sum3(off[0] * off[0], off[1] * off[1], off[2] * off[2]);
  const double s = sqrt(z);
  for (int a = 0; a < 3; ++a) {
    const double nrm = z > 0.0 ? off[a] / s : off[a];
    g[a] = ev_inside(v) ? nrm : -nrm;
  }
}
static void query_point(const vxo_layer* E, const double p[3], int want_gradient, int interp,
                        vxm_query_result* out) { /* query.cpp:64-143 */
  memset(out, 0, sizeof *out);
  if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) return;
  const double vs = E->vs;
  const ev_t* at = esdf_voxel_at(E, (int64_t)floor(p[0] / vs), (int64_t)floor(p[1] / vs),
                                 (int64_t)floor(p[2] / vs));
  if (!at || !ev_observed(at)) return;
  out->known = 1;
  double q[3], fl[3], w[3];
  int64_t base[3];
  for (int a = 0; a < 3; ++a) {
    q[a] = p[a] / vs - 0.5;
    fl[a] = floor(q[a]);
    base[a] = (int64_t)fl[a];
    w[a] = q[a] - fl[a];
    if (w[a] < 1e-6) w[a] = 0.0;
    else if (w[a] > 1.0 - 1e-6) w[a] = 1.0;
  }
  int corners_known = interp;
  double d[2][2][2];
  if (interp) {
    for (int dz = 0; dz < 2 && corners_known; ++dz)
      for (int dy = 0; dy < 2 && corners_known; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          const ev_t* v = esdf_voxel_at(E, base[0] + dx, base[1] + dy, base[2] + dz);
          if (!v || !ev_observed(v)) {
            corners_known = 0;
            break;
          }
          d[dx][dy][dz] = esdf_distance(v, vs);
        }
  }
  if (!corners_known) {
    out->distance = esdf_distance(at, vs);
    if (want_gradient) parent_gradient(at, out->gradient);
    return;
  }
  const double ix = 1.0 - w[0], iy = 1.0 - w[1], iz = 1.0 - w[2];
  out->distance = iz * (iy * (ix * d[0][0][0] + w[0] * d[1][0][0]) +
                        w[1] * (ix * d[0][1][0] + w[0] * d[1][1][0])) +
                  w[2] * (iy * (ix * d[0][0][1] + w[0] * d[1][0][1]) +
                          w[1] * (ix * d[0][1][1] + w[0] * d[1][1][1]));
  if (want_gradient) {
    double g[3];
    g[0] = iz * (iy * (d[1][0][0] - d[0][0][0]) + w[1] * (d[1][1][0] - d[0][1][0])) +
           w[2] * (iy * (d[1][0][1] - d[0][0][1]) + w[1] * (d[1][1][1] - d[0][1][1]));
    g[1] = iz * (ix * (d[0][1][0] - d[0][0][0]) + w[0] * (d[1][1][0] - d[1][0][0])) +
           w[2] * (ix * (d[0][1][1] - d[0][0][1]) + w[0] * (d[1][1][1] - d[1][0][1]));
    g[2] = iy * (ix * (d[0][0][1] - d[0][0][0]) + w[0] * (d[1][0][1] - d[1][0][0])) +
           w[1] * (ix * (d[0][1][1] - d[0][1][0]) + w[0] * (d[1][1][1] - d[1][1][0]));
    const double nrm = sqrt(sum3(g[0] * g[0], g[1] * g[1], g[2] * g[2]));
    if (nrm > 1e-9) {
      for (int a = 0; a < 3; ++a) out->gradient[a] = g[a] / nrm;
    } else {
      parent_gradient(at, out->gradient);
    }
  }
}
int vxo_query_batch(const vxo_layer* esdf, const double* xyz, uint64_t n, int want_gradient,
                    const vxm_query_config* cfg, vxm_query_result* out) {
  for (uint64_t i = 0; i < n; ++i)
    query_point(esdf, xyz + 3 * i, want_gradient, cfg->interpolate, &out[i]);
  return VXM_OK;
}
