"""Python host mirror of the reference's C++ mapper API (namespace ``voxmap``,
/root/reference/proj/include), over the C-ABI of libvoxmap_b200.so.

Names, argument meaning and error behaviour follow the reference:

=====================================  ==============================================
reference (proj/include/voxmap/...)    here
=====================================  ==============================================
Layer<TsdfVoxel>, Layer<EsdfVoxel>,    TsdfLayer, EsdfLayer,       core/layer.hpp:47-125
Layer<OccupancyVoxel>,                 OccupancyLayer, ColorLayer
Layer<ColorVoxel>
integrate_color                        integrate_color             integrate/integrator.hpp:57-66
MeshLayer / mesh_block / update_mesh   MeshLayer / mesh_block /    mesh/marching_cubes.hpp:35-78
/ save_mesh_ply                        update_mesh / save_mesh_ply mesh/ply.hpp:27-29
integrate_depth (camera / lidar;       integrate_depth             integrate/integrator.hpp:36-55
TSDF or occupancy layer)
blocks_in_view                         blocks_in_view              sensor/view.hpp:38-48
update_esdf / mark_sites /             update_esdf / mark_sites /  esdf/integrator.hpp:81-120
clear_invalid / lower_esdf             clear_invalid / lower_esdf
EsdfUpdateState                        EsdfUpdateState             esdf/integrator.hpp:67-74
query_batch                            query_batch                 query/query.hpp:59-62
InvalidPoseError / MapCapacityError /  InvalidPoseError / MapCapacityError / InvalidArgumentError
std::invalid_argument                  (a ValueError)
=====================================  ==============================================

Block lists are ``(N, 3) int32`` numpy arrays of GridIndex in lexicographic
order; voxel blocks are numpy structured arrays (TSDF_DTYPE / ESDF_DTYPE /
OCCUPANCY_DTYPE).  update_esdf / mark_sites take a TSDF or an occupancy source
layer, as the reference's overloads do.
There is no CPU fallback: without a B200 every compute call raises
``VoxmapCudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _abi as A
from ._abi import (Camera as CameraIntrinsics, Lidar as LidarIntrinsics,  # noqa: F401
                   default_camera as default_camera_intrinsics,
                   default_lidar as default_lidar_intrinsics,
                   default_integrator_config as IntegratorConfig,
                   default_esdf_config as EsdfConfig, TSDF_DTYPE, ESDF_DTYPE, QUERY_DTYPE,
                   OCCUPANCY_DTYPE)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libvoxmap_b200.so")
# A/B measurements of kernel variants (tools/ab.py) load another build of the
# same library; it is still the native library, never a fallback.
LIB_PATH = os.environ.get("VXM_LIB_PATH", LIB_PATH)


class VoxmapError(RuntimeError):
    pass


class InvalidPoseError(VoxmapError):
    """voxmap::InvalidPoseError (sensor/pose.hpp:23-26)."""


class MapCapacityError(VoxmapError):
    """voxmap::MapCapacityError (core/layer.hpp:28-31)."""


class InvalidArgumentError(VoxmapError, ValueError):
    """std::invalid_argument."""


class VoxmapCudaError(VoxmapError):
    """No usable sm_100 device / CUDA failure (there is no CPU fallback)."""


class IoError(VoxmapError):
    """voxmap::IoError (core/serialization.hpp:24-27)."""


_ERRORS = {A.VXM_ERR_INVALID_POSE: InvalidPoseError, A.VXM_ERR_INVALID_ARGUMENT: InvalidArgumentError,
           A.VXM_ERR_CAPACITY: MapCapacityError, A.VXM_ERR_CUDA: VoxmapCudaError,
           A.VXM_ERR_INTERNAL: VoxmapError, A.VXM_ERR_IO: IoError}

_lib = None
_lib_lock = threading.Lock()


def lib():
    """Loads libvoxmap_b200.so (fails loudly when it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                                  "(make -C paper_2311_00626_b200)")
            L = C.CDLL(LIB_PATH)
            L.vxm_last_error.restype = C.c_char_p
            L.vxm_version.restype = C.c_char_p
            L.vxm_layer_voxel_size.restype = C.c_double
            L.vxm_context_launch_count.restype = C.c_uint64
            L.vxm_pose_valid.restype = C.c_int
            _lib = L
        return _lib


def check(rc):
    if rc != A.VXM_OK:
        raise _ERRORS.get(rc, VoxmapError)(lib().vxm_last_error().decode())


class Pose:
    """Pose (sensor/pose.hpp:30-60): p_parent = R @ p_child + t."""

    def __init__(self, R=None, t=None):
        self.R = np.eye(3) if R is None else np.asarray(R, dtype=np.float64).reshape(3, 3)
        self.t = np.zeros(3) if t is None else np.asarray(t, dtype=np.float64).reshape(3)

    @staticmethod
    def from_c(p: A.PoseC) -> "Pose":
        R, t = A.pose_arrays(p)
        return Pose(R, t)

    def c(self) -> A.PoseC:
        return A.pose_c(self.R, self.t)

    def valid(self) -> bool:
        return bool(lib().vxm_pose_valid(C.byref(self.c())))

    def inverse(self) -> "Pose":
        o = A.PoseC()
        lib().vxm_pose_inverse(C.byref(self.c()), C.byref(o))
        return Pose.from_c(o)


def _pose_c(T):
    return T.c() if isinstance(T, Pose) else T


class Context:
    """One CUDA device + stream (calls on a context are serialized)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().vxm_context_create(C.c_int(device), C.byref(h)))
        self.h = h
        self.device = device

    def __del__(self):
        try:
            lib().vxm_context_destroy(self.h)
        except Exception:
            pass

    def synchronize(self):
        check(lib().vxm_context_synchronize(self.h))

    def set_shard(self, rank: int, world: int, slab: int = 16):
        check(lib().vxm_context_set_shard(self.h, rank, world, slab))

    @property
    def launch_count(self) -> int:
        return int(lib().vxm_context_launch_count(self.h))

    @property
    def stream(self) -> int:
        """cudaStream_t handle (e.g. for torch.cuda.ExternalStream)."""
        lib().vxm_context_stream.restype = C.c_uint64
        return int(lib().vxm_context_stream(self.h))

    def stats(self) -> dict:
        s = Stats()
        check(lib().vxm_context_stats(self.h, C.byref(s)))
        return {f: int(getattr(s, f)) for f, _ in Stats._fields_ if f != "reserved"} | {
            "esdf_changed_blocks": int(s.reserved[0]), "quiet_blocks": int(s.reserved[1])}

    def reset_stats(self):
        lib().vxm_context_reset_stats(self.h)

    def set_profiling(self, enable: bool):
        check(lib().vxm_context_set_profiling(self.h, C.c_int(int(enable))))

    def kernel_time(self, name: str):
        """(total ms, launches) of one instrumented kernel since the last reset."""
        ms = C.c_double()
        n = C.c_uint64()
        check(lib().vxm_context_kernel_time(self.h, name.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def reset_kernel_times(self):
        lib().vxm_context_reset_kernel_times(self.h)


class Stats(C.Structure):
    """vxm_stats (include/voxmap_b200.h)."""
    _fields_ = [(f, C.c_uint64) for f in (
        "integrate_calls", "candidate_blocks", "new_blocks", "changed_blocks", "voxels_read",
        "voxels_updated", "depth_pixels", "esdf_calls", "esdf_blocks", "effective_blocks",
        "esdf_new_blocks", "lower_rounds", "dirty_blocks_after_round1", "pair_exchanges",
        "compared_blocks")] + [("reserved", C.c_uint64 * 8)]


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("VOXMAP_DEVICE", "0")))
    return _default_ctx


class BlockList:
    """Library-owned std::vector<GridIndex> (device-resident, host on demand)."""

    def __init__(self, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().vxm_blocklist_create(self.ctx.h, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().vxm_blocklist_destroy(self.h)
        except Exception:
            pass

    def numpy(self) -> np.ndarray:
        p = C.c_void_p()
        n = C.c_uint64()
        check(lib().vxm_blocklist_host(self.h, C.byref(p), C.byref(n)))
        return A.keys_array(p, n.value)

    def assign(self, keys):
        k = A.as_keys(keys)
        check(lib().vxm_blocklist_assign(self.h, A.ptr(k), C.c_uint64(len(k))))
        return self


class _Layer:
    kind = None
    dtype = None

    def __init__(self, voxel_size: float, max_blocks: int = 0, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().vxm_layer_create(self.ctx.h, C.c_int(self.kind), C.c_double(voxel_size),
                                     C.c_uint64(max_blocks), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().vxm_layer_destroy(self.h)
        except Exception:
            pass

    def _result_list(self) -> "BlockList":
        """Reused result list (results are copied to numpy immediately)."""
        lst = getattr(self, "_out", None)
        if lst is None:
            lst = self._out = BlockList(self.ctx)
        return lst

    @property
    def voxel_size(self) -> float:
        return float(lib().vxm_layer_voxel_size(self.h))

    @property
    def block_size(self) -> float:
        return self.voxel_size * A.VOXELS_PER_SIDE

    def reserve(self, n_blocks: int) -> None:
        """Pre-size the device pool (vxm_layer_reserve); results are unaffected."""
        check(lib().vxm_layer_reserve(self.h, C.c_uint64(n_blocks)))

    def num_blocks(self) -> int:
        n = C.c_uint64()
        check(lib().vxm_layer_num_blocks(self.h, C.byref(n)))
        return n.value

    def has_blocks(self, keys) -> np.ndarray:
        k = A.as_keys(keys)
        out = np.zeros(len(k), np.uint8)
        check(lib().vxm_layer_has_blocks(self.h, A.ptr(k), C.c_uint64(len(k)), A.ptr(out)))
        return out.astype(bool)

    def has_block(self, g) -> bool:
        return bool(self.has_blocks([g])[0])

    def export(self):
        """(sorted keys (N,3) int32, voxels (N,512) structured)."""
        n = self.num_blocks()
        keys = np.zeros((n, 3), np.int32)
        vox = np.zeros((n, A.VOXELS_PER_BLOCK), self.dtype)
        check(lib().vxm_layer_export(self.h, A.ptr(keys), A.ptr(vox), C.c_uint64(n)))
        return keys, vox

    def sorted_indices(self) -> np.ndarray:
        n = self.num_blocks()
        keys = np.zeros((n, 3), np.int32)
        check(lib().vxm_layer_export(self.h, A.ptr(keys), C.c_void_p(0), C.c_uint64(n)))
        return keys

    def read_blocks(self, keys):
        k = A.as_keys(keys)
        vox = np.zeros((len(k), A.VOXELS_PER_BLOCK), self.dtype)
        found = np.zeros(len(k), np.uint8)
        check(lib().vxm_layer_read_blocks(self.h, A.ptr(k), C.c_uint64(len(k)), A.ptr(vox),
                                          A.ptr(found)))
        return vox, found.astype(bool)

    def block(self, g):
        vox, found = self.read_blocks([g])
        return vox[0] if found[0] else None

    def voxel(self, gv):
        """voxel_ptr (layer.hpp:88-96): the voxel at a global voxel index, or None."""
        blk = self.block(tuple(int(c) for c in block_of_global_voxel(gv)))
        return None if blk is None else blk[int(linear_voxel_index(local_voxel_of_global(gv)))]

    def write_blocks(self, keys, voxels):
        """get_or_allocate + overwrite (host writes through block_ptr)."""
        k = A.as_keys(keys)
        v = np.ascontiguousarray(np.asarray(voxels, self.dtype).reshape(len(k), A.VOXELS_PER_BLOCK))
        check(lib().vxm_layer_write_blocks(self.h, A.ptr(k), C.c_uint64(len(k)), A.ptr(v)))

    def clone(self):
        h = C.c_void_p()
        check(lib().vxm_layer_clone(self.h, C.byref(h)))
        out = object.__new__(type(self))
        out.ctx = self.ctx
        out.h = h
        return out


class TsdfLayer(_Layer):
    kind = A.LAYER_TSDF
    dtype = A.TSDF_DTYPE

    @classmethod
    def _adopt(cls, h, ctx):
        obj = cls.__new__(cls)
        obj.ctx, obj.h = ctx, h
        return obj


class EsdfLayer(_Layer):
    kind = A.LAYER_ESDF
    dtype = A.ESDF_DTYPE

    @classmethod
    def _adopt(cls, h, ctx):
        obj = cls.__new__(cls)
        obj.ctx, obj.h = ctx, h
        return obj


class ColorLayer(_Layer):
    """Layer<ColorVoxel> (core/voxels.hpp:34-41)."""
    kind = A.LAYER_COLOR
    dtype = A.COLOR_DTYPE

    @classmethod
    def _adopt(cls, h, ctx):
        obj = cls.__new__(cls)
        obj.ctx, obj.h = ctx, h
        return obj


class MeshBlock:
    """MeshBlock (mesh/mesh_layer.hpp:16-25): numpy copies of one block's mesh."""

    def __init__(self, vertices, normals, colors, triangles):
        self.vertices, self.normals, self.colors, self.triangles = vertices, normals, colors, triangles

    def empty(self) -> bool:
        return len(self.triangles) == 0


class MeshLayer:
    """MeshLayer (mesh/mesh_layer.hpp:27-66); meshes are computed on the device."""

    def __init__(self, voxel_size: float, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().vxm_mesh_layer_create(self.ctx.h, C.c_double(voxel_size), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().vxm_mesh_layer_destroy(self.h)
        except Exception:
            pass

    @property
    def voxel_size(self) -> float:
        lib().vxm_mesh_layer_voxel_size.restype = C.c_double
        return float(lib().vxm_mesh_layer_voxel_size(self.h))

    def num_blocks(self) -> int:
        lib().vxm_mesh_layer_num_blocks.restype = C.c_uint64
        return int(lib().vxm_mesh_layer_num_blocks(self.h))

    def sorted_indices(self) -> np.ndarray:
        n = self.num_blocks()
        keys = np.zeros((n, 3), np.int32)
        check(lib().vxm_mesh_layer_sorted_indices(self.h, A.ptr(keys), C.c_uint64(n)))
        return keys

    def block(self, g):
        """block_ptr: MeshBlock or None."""
        k = A.as_keys([g])
        v = A.MeshBlockViewC()
        found = C.c_int()
        check(lib().vxm_mesh_layer_block(self.h, A.ptr(k), C.byref(v), C.byref(found)))
        if not found.value:
            return None

        def arr(p, n, dt, w):
            if n == 0:
                return np.zeros((0, w), dt)
            return np.ctypeslib.as_array(p, shape=(n * w,)).reshape(n, w).astype(dt, copy=True)
        return MeshBlock(arr(v.vertices, v.n_vertices, np.float32, 3),
                         arr(v.normals, v.n_vertices, np.float32, 3),
                         arr(v.colors, v.n_colors, np.uint8, 3),
                         arr(v.triangles, v.n_triangles, np.uint32, 3))

    def erase(self, g) -> None:
        check(lib().vxm_mesh_layer_erase(self.h, A.ptr(A.as_keys([g]))))


class HostBuffer:
    """Page-locked host buffer (vxm_host_alloc) viewed as a numpy array: frames
    staged here upload at full PCIe rate through the host-buffer entry points."""

    def __init__(self, shape, dtype=np.float32):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        check(lib().vxm_host_alloc(C.c_uint64(self.nbytes), C.byref(p)))
        self._p = p
        buf = (C.c_ubyte * max(self.nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        try:
            lib().vxm_host_free(self._p)
        except Exception:
            pass


def pinned_like(a):
    """A page-locked copy of array `a` (HostBuffer); keep the buffer alive."""
    hb = HostBuffer(a.shape, a.dtype)
    hb.array[...] = a
    return hb


def _color(rgb):
    c = np.ascontiguousarray(rgb, dtype=np.uint8)
    if c.ndim != 3 or c.shape[2] != 3:
        raise InvalidArgumentError("color image must be (height, width, 3) uint8")
    return c


def integrate_color(color: ColorLayer, rgb, depth, T_LS, camera, tsdf: TsdfLayer, cfg=None,
                    out: BlockList | None = None):
    """integrate_color (integrate/integrator.hpp:57-66): fuses an RGB image
    ((H, W, 3) uint8) into the TSDF surface band; returns the changed blocks."""
    cfg = cfg or IntegratorConfig()
    c, d = _color(rgb), _depth(depth)
    out = out or color._result_list()
    check(lib().vxm_integrate_color(color.h, A.ptr(c), C.c_int(c.shape[1]), C.c_int(c.shape[0]),
                                    A.ptr(d), C.c_int(d.shape[1]), C.c_int(d.shape[0]),
                                    C.byref(_pose_c(T_LS)), C.byref(camera), tsdf.h, C.byref(cfg),
                                    out.h))
    return out.numpy()


def mesh_block(mesh: MeshLayer, tsdf: TsdfLayer, g, cfg=None, color: ColorLayer | None = None):
    """mesh_block (mesh/marching_cubes.hpp:67-69): meshes block g into `mesh`
    (get_or_create(g) = mesh_block(...)) and returns its MeshBlock."""
    cfg = cfg or A.default_mesh_config()
    check(lib().vxm_mesh_block(mesh.h, tsdf.h, A.ptr(A.as_keys([g])), C.byref(cfg),
                               color.h if color is not None else None))
    return mesh.block(g)


def update_mesh(mesh: MeshLayer, tsdf: TsdfLayer, updated, cfg=None, color: ColorLayer | None = None):
    """update_mesh (mesh/marching_cubes.hpp:71-78): returns the re-meshed blocks."""
    cfg = cfg or A.default_mesh_config()
    out = BlockList(mesh.ctx)
    cl = color.h if color is not None else None
    if isinstance(updated, BlockList):
        check(lib().vxm_update_mesh_list(mesh.h, tsdf.h, updated.h, C.byref(cfg), cl, out.h))
    else:
        k = A.as_keys(updated)
        check(lib().vxm_update_mesh(mesh.h, tsdf.h, A.ptr(k), C.c_uint64(len(k)), C.byref(cfg), cl,
                                    out.h))
    return out.numpy()


def save_mesh_ply(mesh: MeshLayer, path: str) -> None:
    """save_mesh_ply (mesh/ply.hpp:27-29)."""
    check(lib().vxm_save_mesh_ply(mesh.h, os.fsencode(path)))


class OccupancyLayer(_Layer):
    """Layer<OccupancyVoxel> (core/voxels.hpp:28-32): log-odds, 0 = unobserved."""
    kind = A.LAYER_OCCUPANCY
    dtype = A.OCCUPANCY_DTYPE

    @classmethod
    def _adopt(cls, h, ctx):
        obj = cls.__new__(cls)
        obj.ctx, obj.h = ctx, h
        return obj


def make_replay_config(voxel_size: float) -> A.ReplayConfigC:
    """make_replay_config (io/pipeline.cpp:46-52)."""
    c = A.ReplayConfigC()
    lib().vxm_replay_config_make(C.c_double(voxel_size), C.byref(c))
    return c


def replay_cake(frames, intrinsics, cfg: A.ReplayConfigC, ctx: Context | None = None):
    """replay (io/pipeline.cpp:54-148) over in-memory frames [(T_WS, depth) or
    (T_WS, depth, rgb), ...] -> (cake, timings): cake is a dict of the layers
    replay created ("source": TsdfLayer / OccupancyLayer, "esdf", "color",
    "mesh"; None when never required) and timings the FrameTiming records
    (FRAME_TIMING_DTYPE)."""
    ctx = ctx or default_context()
    n = len(frames)
    rgb = None
    if n:
        depth = np.ascontiguousarray(np.stack([_depth(f[1]) for f in frames]), np.float32)
        h, w = depth.shape[1], depth.shape[2]
        poses = (A.PoseC * n)(*[_pose_c(f[0]) for f in frames])
        if all(len(f) > 2 and f[2] is not None for f in frames):
            rgb = np.ascontiguousarray(np.stack([_color(f[2]) for f in frames]))
    else:
        depth, h, w, poses = np.zeros((0, 0, 0), np.float32), 0, 0, (A.PoseC * 1)()
    timings = np.zeros(max(n, 1), A.FRAME_TIMING_DTYPE)
    res = A.ReplayResultC()
    if isinstance(intrinsics, A.Camera):
        check(lib().vxm_replay_camera(ctx.h, C.byref(cfg), C.byref(intrinsics), C.c_int(n), C.c_int(w),
                                      C.c_int(h), A.ptr(depth), A.ptr(rgb) if rgb is not None else None,
                                      poses, C.byref(res), A.ptr(timings)))
    else:
        check(lib().vxm_replay_lidar(ctx.h, C.byref(cfg), C.byref(intrinsics), C.c_int(n), C.c_int(w),
                                     C.c_int(h), A.ptr(depth), poses, C.byref(res), A.ptr(timings)))
    src_cls = OccupancyLayer if cfg.use_occupancy else TsdfLayer
    mesh = None
    if res.mesh:
        mesh = MeshLayer.__new__(MeshLayer)
        mesh.ctx, mesh.h = ctx, C.c_void_p(res.mesh)
    cake = {"source": src_cls._adopt(C.c_void_p(res.source), ctx) if res.source else None,
            "esdf": EsdfLayer._adopt(C.c_void_p(res.esdf), ctx) if res.esdf else None,
            "color": ColorLayer._adopt(C.c_void_p(res.color), ctx) if res.color else None,
            "mesh": mesh}
    return cake, timings[:n]


def replay(frames, intrinsics, cfg: A.ReplayConfigC, ctx: Context | None = None):
    """replay (io/pipeline.cpp:54-148) -> (source, esdf, timings); see replay_cake
    for the color and mesh layers."""
    cake, timings = replay_cake(frames, intrinsics, cfg, ctx)
    return cake["source"], cake["esdf"], timings


def write_timing_csv(timings, path: str) -> None:
    """write_timing_csv (io/pipeline.cpp:150-168): frame,tsdf_ms,color_ms,esdf_ms,mesh_ms."""
    try:
        with open(path, "w", newline="") as f:
            f.write("frame,tsdf_ms,color_ms,esdf_ms,mesh_ms\n")
            for t in timings:
                f.write("%d,%.3f,%.3f,%.3f,%.3f\n" % (t["frame"], t["tsdf_ms"], t["color_ms"],
                                                     t["esdf_ms"], t["mesh_ms"]))
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e


def save_snapshot(path: str, voxel_size: float, tsdf: TsdfLayer | None = None,
                  esdf: EsdfLayer | None = None, occupancy: OccupancyLayer | None = None,
                  color: ColorLayer | None = None) -> None:
    """save_snapshot (core/serialization.hpp:31): VXLF v1, byte-identical to the
    reference's for equal maps (layers tsdf, occupancy, color, esdf)."""
    h = lambda L: L.h if L is not None else None  # noqa: E731
    check(lib().vxm_snapshot_save_layers(os.fsencode(path), C.c_double(voxel_size), h(tsdf),
                                         h(occupancy), h(color), h(esdf)))


def load_snapshot(path: str, ctx: Context | None = None, with_occupancy: bool = False,
                  with_color: bool = False):
    """load_snapshot (core/serialization.hpp:35) -> (voxel_size, tsdf | None, esdf | None);
    with_occupancy / with_color insert the occupancy / color layer before the ESDF:
    (voxel_size, tsdf, [occupancy,] [color,] esdf)."""
    ctx = ctx or default_context()
    vs = C.c_double()
    th, oh, ch, eh = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    check(lib().vxm_snapshot_load_layers(ctx.h, os.fsencode(path), C.byref(vs), C.byref(th),
                                         C.byref(oh) if with_occupancy else None,
                                         C.byref(ch) if with_color else None, C.byref(eh)))
    out = [vs.value, TsdfLayer._adopt(th, ctx) if th.value else None]
    if with_occupancy:
        out.append(OccupancyLayer._adopt(oh, ctx) if oh.value else None)
    if with_color:
        out.append(ColorLayer._adopt(ch, ctx) if ch.value else None)
    out.append(EsdfLayer._adopt(eh, ctx) if eh.value else None)
    return tuple(out)


def _depth(depth):
    d = np.ascontiguousarray(depth, dtype=np.float32)
    if d.ndim != 2:
        raise InvalidArgumentError("depth image must be 2-D (height, width)")
    return d


def integrate_depth(layer, depth, T_LS, intrinsics, cfg=None, out: BlockList | None = None):
    """integrate_depth (integrate/integrator.hpp:36-55): fuses one frame into a
    TsdfLayer (tsdf_update) or an OccupancyLayer (occupancy_update) and returns
    the sorted indices of the blocks whose bytes changed."""
    cfg = cfg or IntegratorConfig()
    d = _depth(depth)
    out = out or layer._result_list()
    fn = (lib().vxm_integrate_depth_camera if isinstance(intrinsics, A.Camera)
          else lib().vxm_integrate_depth_lidar)
    check(fn(layer.h, A.ptr(d), C.c_int(d.shape[1]), C.c_int(d.shape[0]), C.byref(_pose_c(T_LS)),
             C.byref(intrinsics), C.byref(cfg), out.h))
    return out.numpy()


def integrate_depth_device(layer: TsdfLayer, depth_dev_ptr: int, width: int, height: int, T_LS,
                           intrinsics, cfg, out: BlockList) -> BlockList:
    """Device-resident variant (depth already in HBM; changed list stays on device)."""
    fn = (lib().vxm_integrate_depth_camera_device if isinstance(intrinsics, A.Camera)
          else lib().vxm_integrate_depth_lidar_device)
    check(fn(layer.h, C.c_void_p(depth_dev_ptr), C.c_int(width), C.c_int(height),
             C.byref(_pose_c(T_LS)), C.byref(intrinsics), C.byref(cfg), out.h))
    return out


def diag_lidar_angles(xyz, ctx: Context | None = None):
    """(azimuth, polar) of sensor-frame points exactly as the LiDAR integration
    computes them on the device (lidar.hpp:43-55): atan2(y, x) and
    acos(z / |p|).  Diagnostics for the parity tests."""
    ctx = ctx or default_context()
    p = np.ascontiguousarray(np.asarray(xyz, np.float64).reshape(-1, 3))
    az = np.empty(len(p), np.float64)
    po = np.empty(len(p), np.float64)
    check(lib().vxm_diag_lidar_angles(ctx.h, A.ptr(p), C.c_uint64(len(p)), A.ptr(az), A.ptr(po)))
    return az, po


def blocks_in_view(T_LS, intrinsics, depth, block_size, cfg=None, ctx: Context | None = None):
    """blocks_in_view (sensor/view.hpp:38-48): sorted unique candidate blocks."""
    ctx = ctx or default_context()
    cfg = cfg or A.ViewConfigC(5.0, 0.2, 8)
    d = _depth(depth)
    out = BlockList(ctx)
    fn = (lib().vxm_blocks_in_view_camera if isinstance(intrinsics, A.Camera)
          else lib().vxm_blocks_in_view_lidar)
    check(fn(ctx.h, C.byref(_pose_c(T_LS)), C.byref(intrinsics), A.ptr(d), C.c_int(d.shape[1]),
             C.c_int(d.shape[0]), C.c_double(block_size), C.byref(cfg), out.h))
    return out.numpy()


def update_esdf(esdf: EsdfLayer, tsdf, updated, cfg=None, out: BlockList | None = None):
    """update_esdf (esdf/integrator.hpp:113-120) from a TsdfLayer or an
    OccupancyLayer source. `updated` may be a BlockList (e.g. the
    device-resident output of integrate_depth) or an (N,3) array."""
    cfg = cfg or EsdfConfig()
    out = out or esdf._result_list()
    if isinstance(updated, BlockList):
        check(lib().vxm_update_esdf_list(esdf.h, tsdf.h, updated.h, C.byref(cfg), out.h))
    else:
        k = A.as_keys(updated)
        check(lib().vxm_update_esdf(esdf.h, tsdf.h, A.ptr(k), C.c_uint64(len(k)), C.byref(cfg),
                                    out.h))
    return out.numpy()


def update_esdf_sharded(esdf_shards, tsdf_shards, updated, cfg, out=None):
    """update_esdf over a block-sharded map (vxm_update_esdf_sharded): shard p's
    context must be set_shard(p, P, slab); `updated[p]` is shard p's changed list
    (BlockList or (N,3) array).  Returns the per-shard changed lists."""
    P = len(esdf_shards)
    lists = []
    for p in range(P):
        u = updated[p]
        if not isinstance(u, BlockList):
            bl = BlockList(esdf_shards[p].ctx)
            bl.assign(u)
            u = bl
        lists.append(u)
    out = out or [BlockList(esdf_shards[p].ctx) for p in range(P)]
    arr = lambda xs: (C.c_void_p * P)(*[x.h.value for x in xs])  # noqa: E731
    check(lib().vxm_update_esdf_sharded(C.c_int(P), arr(esdf_shards), arr(tsdf_shards), arr(lists),
                                        C.byref(cfg), arr(out)))
    return [o.numpy() for o in out]


def update_esdf_device(esdf: EsdfLayer, tsdf: TsdfLayer, updated: BlockList, cfg,
                       out: BlockList) -> BlockList:
    """Device-resident update_esdf: consumes and produces device block lists."""
    check(lib().vxm_update_esdf_list(esdf.h, tsdf.h, updated.h, C.byref(cfg), out.h))
    return out


def update_frame_device(tsdf: TsdfLayer, esdf: EsdfLayer | None, depth_dev_ptr: int, width: int,
                        height: int, T_LS, intrinsics, icfg, ecfg, tsdf_out: BlockList,
                        esdf_out: BlockList | None) -> None:
    """One replay-pipeline frame (pipeline.cpp:95-108): integrate_depth then
    update_esdf on a device-resident depth image with one host round trip;
    both changed lists stay on the device.  `esdf=None` integrates only."""
    fn = (lib().vxm_update_frame_camera_device if isinstance(intrinsics, A.Camera)
          else lib().vxm_update_frame_lidar_device)
    check(fn(tsdf.h, esdf.h if esdf is not None else None, C.c_void_p(depth_dev_ptr),
             C.c_int(width), C.c_int(height), C.byref(_pose_c(T_LS)), C.byref(intrinsics),
             C.byref(icfg), C.byref(ecfg) if ecfg is not None else None, tsdf_out.h,
             esdf_out.h if esdf_out is not None else None))


class EsdfUpdateState:
    """EsdfUpdateState (esdf/integrator.hpp:67-74)."""

    def __init__(self):
        h = C.c_void_p()
        check(lib().vxm_esdf_state_create(C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().vxm_esdf_state_destroy(self.h)
        except Exception:
            pass

    def _get(self, which):
        p = C.c_void_p()
        n = C.c_uint64()
        check(lib().vxm_esdf_state_get(self.h, C.c_int(which), C.byref(p), C.byref(n)))
        return A.keys_array(p, n.value)

    def _set(self, which, keys):
        k = A.as_keys(keys)
        check(lib().vxm_esdf_state_set(self.h, C.c_int(which), A.ptr(k), C.c_uint64(len(k))))

    indices_to_update = property(lambda s: s._get(0), lambda s, v: s._set(0, v))
    indices_to_clear = property(lambda s: s._get(1), lambda s, v: s._set(1, v))
    cleared_indices = property(lambda s: s._get(2), lambda s, v: s._set(2, v))


def mark_sites(esdf, tsdf, updated, cfg, state: EsdfUpdateState):
    k = A.as_keys(updated)
    out = BlockList(esdf.ctx)
    check(lib().vxm_esdf_mark_sites(esdf.h, tsdf.h, A.ptr(k), C.c_uint64(len(k)), C.byref(cfg),
                                    state.h, out.h))
    return out.numpy()


def clear_invalid(esdf, cfg, state: EsdfUpdateState):
    out = BlockList(esdf.ctx)
    check(lib().vxm_esdf_clear_invalid(esdf.h, C.byref(cfg), state.h, out.h))
    return out.numpy()


def lower_esdf(esdf, state: EsdfUpdateState, cfg):
    """Returns (rounds, changed)."""
    out = BlockList(esdf.ctx)
    rounds = C.c_int()
    check(lib().vxm_esdf_lower(esdf.h, state.h, C.byref(cfg), out.h, C.byref(rounds)))
    return rounds.value, out.numpy()


def query_batch(esdf: EsdfLayer, points, want_gradient: bool = False, interpolate: bool = True):
    """query_batch (query/query.hpp:59-62): structured array (known, distance, gradient)."""
    x = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 3))
    out = np.zeros(len(x), A.QUERY_DTYPE)
    cfg = A.QueryConfigC(int(interpolate), 1)
    check(lib().vxm_query_batch(esdf.h, A.ptr(x), C.c_uint64(len(x)), C.c_int(int(want_gradient)),
                                C.byref(cfg), A.ptr(out)))
    return out


# ---- index algebra (core/indexing.hpp:33-139), vectorised --
def linear_voxel_index(v):
    """x-fastest index inside a block: x + 8 (y + 8 z); v: (..., 3) ints."""
    v = np.asarray(v)
    return v[..., 0] + A.VOXELS_PER_SIDE * (v[..., 1] + A.VOXELS_PER_SIDE * v[..., 2])


def voxel_index_from_linear(lin):
    lin = np.asarray(lin)
    n = A.VOXELS_PER_SIDE
    return np.stack([lin % n, (lin // n) % n, lin // (n * n)], axis=-1)


def global_voxel_index(g, v):
    return np.asarray(g, np.int64) * A.VOXELS_PER_SIDE + np.asarray(v, np.int64)


def block_of_global_voxel(gv):
    """floor(gv / 8) per axis (floor_div_side, correct for negatives)."""
    return np.floor_divide(np.asarray(gv, np.int64), A.VOXELS_PER_SIDE).astype(np.int32)


def local_voxel_of_global(gv):
    return np.mod(np.asarray(gv, np.int64), A.VOXELS_PER_SIDE).astype(np.int32)


def position_to_global_voxel(p, voxel_size):
    """floor(p / voxel_size) per axis (indexing.hpp:96-102)."""
    return np.floor(np.asarray(p, np.float64) / voxel_size).astype(np.int64)


def position_to_indices(p, voxel_size):
    """(block index, voxel index) containing metric position(s) p."""
    gv = position_to_global_voxel(p, voxel_size)
    return block_of_global_voxel(gv), local_voxel_of_global(gv)


def voxel_center(g, v, voxel_size):
    """((8 g + v) + 0.5) * voxel_size, the reference's association (indexing.hpp:113-119)."""
    return ((np.asarray(g, np.float64) * A.VOXELS_PER_SIDE + np.asarray(v)) + 0.5) * voxel_size


def block_origin(g, voxel_size):
    return np.asarray(g, np.float64) * (A.VOXELS_PER_SIDE * voxel_size)


def esdf_distance(sq, inside, voxel_size):
    """esdf_distance (esdf/integrator.hpp:59-63)."""
    d = np.sqrt(np.asarray(sq, np.float64)) * voxel_size
    return np.where(inside, -d, d)
