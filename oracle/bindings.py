"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the two CPU oracles.

* ``PortOracle``  -> oracle/_lib/libvoxmap_oracle.so (plain-C restatement,
  oracle/voxmap_oracle.c).
* ``RefOracle``   -> oracle/_ref/libvoxmap_ref.so (the reference's own sources
  compiled against oracle/eigen_shim, driven by oracle/ref_driver.cpp).

Both expose the same small interface so tests can run either as the checker.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2311_00626_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_lib", "libvoxmap_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libvoxmap_ref.so")


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Base:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        p = self.prefix
        self._f = lambda name: getattr(self.lib, p + name)
        self._f("last_error").restype = C.c_char_p
        self._f("layer_num_blocks").restype = C.c_uint64

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._f("last_error")().decode())

    def _list(self, call, *args):
        out = C.c_void_p()
        n = C.c_uint64()
        self._check(call(*args, C.byref(out), C.byref(n)))
        keys = A.keys_array(out, n.value)
        self._f("free")(out)
        return keys

    # --- layers ----------------------------------------------------------
    def layer(self, kind, voxel_size, max_blocks=0):
        h = C.c_void_p()
        self._check(self._f("layer_create")(C.c_int(kind), C.c_double(voxel_size),
                                            C.c_uint64(max_blocks), C.byref(h)))
        return OracleLayer(self, h, kind, voxel_size)

    def export(self, layer):
        n = int(self._f("layer_num_blocks")(layer.h))
        keys = np.zeros((n, 3), np.int32)
        dt = A.layer_dtype(layer.kind)
        vox = np.zeros((n, 512), dt)
        self._check(self._f("layer_export")(layer.h, A.ptr(keys), A.ptr(vox)))
        return keys, vox

    def write_blocks(self, layer, keys, voxels):
        keys = A.as_keys(keys)
        vox = np.ascontiguousarray(voxels)
        self._check(self._f("layer_write_blocks")(layer.h, A.ptr(keys), C.c_uint64(len(keys)),
                                                  A.ptr(vox)))

    # --- hot path ---------------------------------------------------------
    def blocks_in_view_camera(self, T, cam, depth, block_size, vcfg):
        d = np.ascontiguousarray(depth, np.float32)
        return self._list(self._f("blocks_in_view_camera"), C.byref(T), C.byref(cam), A.ptr(d),
                          C.c_int(d.shape[1]), C.c_int(d.shape[0]), C.c_double(block_size),
                          C.byref(vcfg))

    def blocks_in_view_lidar(self, T, li, depth, block_size, vcfg):
        d = np.ascontiguousarray(depth, np.float32)
        return self._list(self._f("blocks_in_view_lidar"), C.byref(T), C.byref(li), A.ptr(d),
                          C.c_int(d.shape[1]), C.c_int(d.shape[0]), C.c_double(block_size),
                          C.byref(vcfg))

    def update_esdf(self, esdf, tsdf, updated, cfg):
        u = A.as_keys(updated)
        return self._list(self._f("update_esdf"), esdf.h, tsdf.h, A.ptr(u), C.c_uint64(len(u)),
                          C.byref(cfg))

    def state(self):
        return OracleState(self)

    def mark_sites(self, esdf, tsdf, updated, cfg, st):
        u = A.as_keys(updated)
        return self._list(self._f("mark_sites"), esdf.h, tsdf.h, A.ptr(u), C.c_uint64(len(u)),
                          C.byref(cfg), st.h)

    def clear_invalid(self, esdf, cfg, st):
        return self._list(self._f("clear_invalid"), esdf.h, C.byref(cfg), st.h)

    def lower_esdf(self, esdf, st, cfg):
        rounds = C.c_int()
        out = C.c_void_p()
        n = C.c_uint64()
        self._check(self._f("lower_esdf")(esdf.h, st.h, C.byref(cfg), C.byref(rounds),
                                          C.byref(out), C.byref(n)))
        keys = A.keys_array(out, n.value)
        self._f("free")(out)
        return rounds.value, keys


class OracleLayer:
    def __init__(self, owner, h, kind, vs):
        self.owner, self.h, self.kind, self.voxel_size = owner, h, kind, vs

    def __del__(self):
        try:
            self.owner._f("layer_destroy")(self.h)
        except Exception:
            pass

    @property
    def num_blocks(self):
        return int(self.owner._f("layer_num_blocks")(self.h))

    def export(self):
        return self.owner.export(self)


class OracleMesh:
    """voxmap_ref::MeshLayer handle; block(g) -> (vertices, normals, colors, triangles)."""

    def __init__(self, owner, vs):
        self.owner = owner
        owner.lib.vxr_mesh_create.restype = C.c_void_p
        owner.lib.vxr_mesh_num_blocks.restype = C.c_uint64
        self.h = C.c_void_p(owner.lib.vxr_mesh_create(C.c_double(vs)))

    def __del__(self):
        try:
            self.owner.lib.vxr_mesh_destroy(self.h)
        except Exception:
            pass

    def sorted_indices(self):
        n = int(self.owner.lib.vxr_mesh_num_blocks(self.h))
        keys = np.zeros((n, 3), np.int32)
        self.owner.lib.vxr_mesh_keys(self.h, A.ptr(keys))
        return keys

    def block(self, g):
        k = A.as_keys([g])
        nv, nt, nc = C.c_uint64(), C.c_uint64(), C.c_uint64()
        pv, pn, pt = C.POINTER(C.c_float)(), C.POINTER(C.c_float)(), C.POINTER(C.c_uint32)()
        pc = C.POINTER(C.c_uint8)()
        self.owner._check(self.owner.lib.vxr_mesh_block_get(
            self.h, A.ptr(k), C.byref(nv), C.byref(nt), C.byref(pv), C.byref(pn), C.byref(pc),
            C.byref(nc), C.byref(pt)))

        def arr(p, n, dt):
            if n == 0:
                return np.zeros((0, 3), dt)
            return np.ctypeslib.as_array(p, shape=(3 * n,)).reshape(n, 3).astype(dt, copy=True)
        return (arr(pv, nv.value, np.float32), arr(pn, nv.value, np.float32),
                arr(pc, nc.value, np.uint8), arr(pt, nt.value, np.uint32))


class OracleState:
    def __init__(self, owner):
        self.owner = owner
        owner._f("state_create").restype = C.c_void_p
        self.h = C.c_void_p(owner._f("state_create")())

    def __del__(self):
        try:
            self.owner._f("state_destroy")(self.h)
        except Exception:
            pass

    def get(self, which):
        return self.owner._list(self.owner._f("state_get"), self.h, C.c_int(which))

    def set(self, which, keys):
        k = A.as_keys(keys)
        self.owner._check(self.owner._f("state_set")(self.h, C.c_int(which), A.ptr(k),
                                                     C.c_uint64(len(k))))


class PortOracle(_Base):
    """The plain-C restatement (oracle/voxmap_oracle.c)."""
    prefix = "vxo_"

    def __init__(self, path=PORT_LIB):
        super().__init__(path)

    def integrate_camera(self, layer, depth, T, cam, cfg):
        d = np.ascontiguousarray(depth, np.float32)
        return self._list(self._f("integrate_camera"), layer.h, A.ptr(d), C.c_int(d.shape[1]),
                          C.c_int(d.shape[0]), C.byref(T), C.byref(cam), C.byref(cfg))

    def integrate_lidar(self, layer, depth, T, li, cfg):
        d = np.ascontiguousarray(depth, np.float32)
        return self._list(self._f("integrate_lidar"), layer.h, A.ptr(d), C.c_int(d.shape[1]),
                          C.c_int(d.shape[0]), C.byref(T), C.byref(li), C.byref(cfg))

    def query_batch(self, esdf, xyz, want_gradient, qcfg):
        x = np.ascontiguousarray(np.asarray(xyz, np.float64).reshape(-1, 3))
        out = np.zeros(len(x), A.QUERY_DTYPE)
        self._check(self.lib.vxo_query_batch(esdf.h, A.ptr(x), C.c_uint64(len(x)),
                                             C.c_int(int(want_gradient)), C.byref(qcfg), A.ptr(out)))
        return out

    def pose_valid(self, T):
        return bool(self.lib.vxo_pose_valid(C.byref(T)))

    def pose_inverse(self, T):
        o = A.PoseC()
        self.lib.vxo_pose_inverse(C.byref(T), C.byref(o))
        return o


class RefOracle(_Base):
    """The reference's own sources (oracle/_ref)."""
    prefix = "vxr_"

    def __init__(self, path=REF_LIB):
        super().__init__(path)

    def integrate_camera(self, layer, depth, T, cam, cfg, serial=False):
        d = np.ascontiguousarray(depth, np.float32)
        return self._list(self._f("integrate_camera"), layer.h, A.ptr(d), C.c_int(d.shape[1]),
                          C.c_int(d.shape[0]), C.byref(T), C.byref(cam), C.byref(cfg),
                          C.c_int(int(serial)))

    def integrate_lidar(self, layer, depth, T, li, cfg, serial=False):
        d = np.ascontiguousarray(depth, np.float32)
        return self._list(self._f("integrate_lidar"), layer.h, A.ptr(d), C.c_int(d.shape[1]),
                          C.c_int(d.shape[0]), C.byref(T), C.byref(li), C.byref(cfg),
                          C.c_int(int(serial)))

    def query_batch(self, esdf, xyz, want_gradient, qcfg, serial=False):
        x = np.ascontiguousarray(np.asarray(xyz, np.float64).reshape(-1, 3))
        out = np.zeros(len(x), A.QUERY_DTYPE)
        self._check(self.lib.vxr_query_batch(esdf.h, A.ptr(x), C.c_uint64(len(x)),
                                             C.c_int(int(want_gradient)), C.byref(qcfg),
                                             C.c_int(int(serial)), A.ptr(out)))
        return out

    def save_snapshot(self, path, voxel_size, tsdf=None, esdf=None, occupancy=None, color=None):
        h = lambda L: L.h if L is not None else None  # noqa: E731
        self._check(self.lib.vxr_snapshot_save(os.fsencode(path), C.c_double(voxel_size),
                                               h(tsdf), h(occupancy), h(color), h(esdf)))

    def load_snapshot(self, path, with_occupancy=False, with_color=False):
        """(vs, tsdf, [occupancy,] [color,] esdf)."""
        vs = C.c_double()
        th, oh, ch, eh = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._check(self.lib.vxr_snapshot_load(os.fsencode(path), C.byref(vs), C.byref(th),
                                               C.byref(oh), C.byref(ch), C.byref(eh)))
        mk = lambda h, kind: OracleLayer(self, h, kind, vs.value) if h.value else None  # noqa: E731
        out = [vs.value, mk(th, A.LAYER_TSDF)]
        if with_occupancy:
            out.append(mk(oh, A.LAYER_OCCUPANCY))
        if with_color:
            out.append(mk(ch, A.LAYER_COLOR))
        out.append(mk(eh, A.LAYER_ESDF))
        return tuple(out)

    # --- color + meshing (integrator.cpp:191-273, marching_cubes.cpp, ply.cpp) ---
    def integrate_color(self, color, rgb, depth, T, cam, tsdf, cfg):
        c = np.ascontiguousarray(rgb, np.uint8)
        d = np.ascontiguousarray(depth, np.float32)
        return self._list(self.lib.vxr_integrate_color, color.h, A.ptr(c), C.c_int(c.shape[1]),
                          C.c_int(c.shape[0]), A.ptr(d), C.byref(T), C.byref(cam), tsdf.h,
                          C.byref(cfg))

    def render_color(self, scene, T, cam):
        out = np.zeros((cam.height, cam.width, 3), np.uint8)
        self._check(self.lib.vxr_render_color_camera(scene.encode(), C.byref(T), C.byref(cam),
                                                     A.ptr(out)))
        return out

    def mc_tri_table(self):
        self.lib.vxr_mc_tri_table.restype = C.POINTER(C.c_int8)
        p = self.lib.vxr_mc_tri_table()
        return np.array([p[i] for i in range(256 * 16)], np.int8).reshape(256, 16)

    def mesh_layer(self, voxel_size):
        return OracleMesh(self, voxel_size)

    def update_mesh(self, mesh, tsdf, updated, min_weight=1e-4, color=None):
        u = A.as_keys(updated)
        return self._list(self.lib.vxr_update_mesh, mesh.h, tsdf.h, A.ptr(u), C.c_uint64(len(u)),
                          C.c_float(min_weight), color.h if color is not None else None)

    def mesh_block(self, mesh, tsdf, g, min_weight=1e-4, color=None):
        k = A.as_keys([g])
        self._check(self.lib.vxr_mesh_block(mesh.h, tsdf.h, A.ptr(k), C.c_float(min_weight),
                                            color.h if color is not None else None))
        return mesh.block(g)

    def save_mesh_ply(self, mesh, path):
        self._check(self.lib.vxr_save_mesh_ply(mesh.h, os.fsencode(path)))

    def orbit_pose(self, scene, k, total, lidar=False):
        p = A.PoseC()
        self._check(self.lib.vxr_orbit_pose(scene.encode(), C.c_int(int(lidar)), C.c_int(k),
                                            C.c_int(total), C.byref(p)))
        return p

    def render_camera(self, scene, T, cam):
        out = np.zeros((cam.height, cam.width), np.float32)
        self._check(self.lib.vxr_render_depth_camera(scene.encode(), C.byref(T), C.byref(cam),
                                                     A.ptr(out)))
        return out

    def render_lidar(self, scene, T, li):
        out = np.zeros((li.num_elevation, li.num_azimuth), np.float32)
        self._check(self.lib.vxr_render_depth_lidar(scene.encode(), C.byref(T), C.byref(li),
                                                    A.ptr(out)))
        return out

    def pose_valid(self, T):
        return bool(self.lib.vxr_pose_valid(C.byref(T)))

    def sphere_world(self, side, vs, trunc, seed=2311, n_spheres=6):
        """Dense C5 TSDF built by ref_driver.cpp (keys (nb^3,3), voxels (nb^3,512))."""
        nb = side // 8
        keys = np.zeros((nb ** 3, 3), np.int32)
        vox = np.zeros((nb ** 3, A.VOXELS_PER_BLOCK), A.TSDF_DTYPE)
        self._check(self.lib.vxr_sphere_world(C.c_int(side), C.c_double(vs), C.c_double(trunc),
                                              C.c_uint(seed), C.c_int(n_spheres), A.ptr(keys),
                                              A.ptr(vox)))
        return keys, vox

    def brute_force_esdf(self, esdf, cfg):
        h = C.c_void_p()
        self._check(self.lib.vxr_brute_force_esdf(esdf.h, C.byref(cfg), C.byref(h)))
        return OracleLayer(self, h, A.LAYER_ESDF, esdf.voxel_size)

    def compare_esdf(self, a, b):
        stats = (C.c_uint64 * 4)()
        mx = C.c_double()
        self._check(self.lib.vxr_compare_esdf(a.h, b.h, stats, C.byref(mx)))
        return dict(compared=stats[0], exact=stats[1], within_one_voxel=stats[2],
                    flag_mismatches=stats[3], max_abs_error=mx.value)


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


def have_port() -> bool:
    return os.path.exists(PORT_LIB)
