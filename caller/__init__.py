"""The stand-in CALLER of the drop-in boundary (not the product).

The reference keeps loading and formatting on the host:
load_hand, load_mesh, sample_surface, decompose_patches, parse_config,
write_dataset.  A production caller uses the reference's own functions for
them; the bench and the tests use this module instead:

* hands come from assets/prepared/<hand>.hand.npz — the reference's own
  load_hand + dependency_groups output, written once by
  tools/prepare_hands.py — so no URDF parser or convex-hull code exists here;
* meshes, surface sampling, host patches, configs and the JSONL writer are
  restated in caller/*.cpp (libgraspgen_caller.so).

Everything handed to libgraspgen_b200.so is a flat lg.h descriptor.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2511_07418_b200 import lgabi as A

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "libgraspgen_caller.so")
PREPARED = os.path.join(ROOT, "assets", "prepared")
_LIB = None


class VisualDesc(C.Structure):
    _fields_ = [("n_links", C.c_int), ("vert_off", A.ip), ("verts", A.dp), ("tri_off", A.ip),
                ("tris", A.ip)]


class LoadReport(C.Structure):
    _fields_ = [("triangles_read", C.c_longlong), ("triangles_kept", C.c_longlong),
                ("degenerate_dropped", C.c_longlong)]


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        import subprocess
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    L = C.CDLL(LIB_PATH)
    vp, P = C.c_void_p, C.POINTER
    sig = {
        "lgc_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
        "lgc_run_params_default": (None, [P(A.RunParams)]),
        "lgc_config_parse": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                       P(C.c_longlong), P(C.c_int), P(C.c_int), P(A.RunParams)]),
        "lgc_index_cache_key": (C.c_int, [P(A.RunParams), P(C.c_uint64)]),
        "lgc_mesh_load": (C.c_int, [C.c_char_p, P(LoadReport), P(vp)]),
        "lgc_mesh_box": (C.c_int, [C.c_double, C.c_double, C.c_double, P(vp)]),
        "lgc_mesh_icosphere": (C.c_int, [C.c_double, C.c_int, P(vp)]),
        "lgc_mesh_cylinder": (C.c_int, [C.c_double, C.c_double, C.c_int, P(vp)]),
        "lgc_mesh_from_arrays": (C.c_int, [A.dp, C.c_int, A.ip, C.c_int, P(vp)]),
        "lgc_mesh_scale": (C.c_int, [vp, C.c_double]),
        "lgc_mesh_info": (C.c_int, [vp, A.ip, A.ip, A.dp]),
        "lgc_mesh_arrays": (C.c_int, [vp, P(A.dp), P(A.ip)]),
        "lgc_mesh_save_obj": (C.c_int, [vp, C.c_char_p]),
        "lgc_mesh_destroy": (None, [vp]),
        "lgc_sample_surface": (C.c_int, [vp, C.c_double, C.c_uint64, A.dp, C.c_size_t,
                                         P(C.c_size_t)]),
        "lgc_hand_patches": (C.c_int, [P(A.HandDesc), P(VisualDesc), C.c_double, C.c_double,
                                       C.c_uint64, C.c_int, P(vp)]),
        "lgc_patches_export": (C.c_int, [vp, P(A.PatchesDesc)]),
        "lgc_patches_destroy": (None, [vp]),
        "lgc_write_dataset": (C.c_int, [C.c_char_p, P(A.Grasp), C.c_longlong]),
        "lgc_write_profile": (C.c_int, [C.c_char_p, P(A.Profile)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


class CallerError(RuntimeError):
    pass


def check(rc):
    if rc != 0:
        buf = C.create_string_buffer(2048)
        lib().lgc_last_error(buf, len(buf))
        msg = buf.value.decode()
        if rc == A.LG_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == A.LG_ERR_OUT_OF_RANGE:
            raise IndexError(msg)
        raise CallerError(msg)


def _dp(a):
    return a.ctypes.data_as(A.dp)


def _ip(a):
    return a.ctypes.data_as(A.ip)


def mix_seed(seed, a, b=0):
    """mix_seed (rng.hpp:25-28), computed in Python (splitmix64)."""
    M = (1 << 64) - 1

    def mix64(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D9B9B3F794A2E5) & M
        return x ^ (x >> 31)

    return mix64(mix64(seed ^ mix64(a)) ^ mix64(b ^ 0x5851F42D4C957F2D))


# ------------------------------------------------------------------ meshes
class Mesh:
    """TriMesh (mesh.hpp:13-21) held by the caller library."""

    def __init__(self, handle, report=None):
        self._h = handle if isinstance(handle, C.c_void_p) else C.c_void_p(handle)
        self.report = report

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.lgc_mesh_destroy(self._h)
            self._h = None

    @staticmethod
    def _make(fn, *args):
        h = C.c_void_p()
        check(fn(*args, C.byref(h)))
        return Mesh(h)

    @classmethod
    def box(cls, size):
        return cls._make(lib().lgc_mesh_box, *map(float, size))

    @classmethod
    def icosphere(cls, radius, subdivisions):
        return cls._make(lib().lgc_mesh_icosphere, float(radius), int(subdivisions))

    @classmethod
    def cylinder(cls, radius, length, segments=24):
        return cls._make(lib().lgc_mesh_cylinder, float(radius), float(length), int(segments))

    @classmethod
    def from_arrays(cls, verts, tris):
        v = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(tris, dtype=np.int32).reshape(-1, 3)
        return cls._make(lib().lgc_mesh_from_arrays, _dp(v), len(v), _ip(t), len(t))

    def info(self):
        nv, nt, area = C.c_int(), C.c_int(), C.c_double()
        check(lib().lgc_mesh_info(self._h, C.byref(nv), C.byref(nt), C.byref(area)))
        return nv.value, nt.value, area.value

    def arrays(self):
        nv, nt, _ = self.info()
        v, t = A.dp(), A.ip()
        check(lib().lgc_mesh_arrays(self._h, C.byref(v), C.byref(t)))
        verts = np.ctypeslib.as_array(v, shape=(nv * 3,)).reshape(nv, 3).copy() if nv else np.zeros((0, 3))
        tris = np.ctypeslib.as_array(t, shape=(nt * 3,)).reshape(nt, 3).copy() if nt else \
            np.zeros((0, 3), np.int32)
        return verts, tris

    def scale(self, s):
        check(lib().lgc_mesh_scale(self._h, float(s)))
        return self

    def save_obj(self, path):
        check(lib().lgc_mesh_save_obj(self._h, str(path).encode()))


def load_mesh(path):
    """load_mesh (mesh.cpp:161-167) with its LoadReport."""
    rep = LoadReport()
    h = C.c_void_p()
    check(lib().lgc_mesh_load(str(path).encode(), C.byref(rep), C.byref(h)))
    return Mesh(h, dict(triangles_read=rep.triangles_read, triangles_kept=rep.triangles_kept,
                        degenerate_dropped=rep.degenerate_dropped))


def sample_surface(mesh, samples_per_cm2, seed):
    """sample_surface (mesh.cpp:297-339) -> float64 array (n, 6) = (p, n)."""
    L = lib()
    n = C.c_size_t()
    check(L.lgc_sample_surface(mesh._h, float(samples_per_cm2), C.c_uint64(seed), None, 0,
                               C.byref(n)))
    out = np.zeros((n.value, 6), dtype=np.float64)
    check(L.lgc_sample_surface(mesh._h, float(samples_per_cm2), C.c_uint64(seed), _dp(out),
                               n.value, C.byref(n)))
    return out


# -------------------------------------------------------------------- hand
class HandModel:
    """The reference's HandModel (hand.hpp:37-46) from its prepared fixture:
    the flat lg_hand_desc, the visual meshes (lg_visual_desc), link and joint
    names and the dependency groups (hand.cpp:374-411)."""

    _ARRAYS = ("parent", "joint_type", "joint_index", "topo_order", "origin_R", "origin_t", "axis",
               "limit_lo", "limit_hi", "part_link", "part_vert_off", "part_verts", "part_tri_off",
               "part_tris", "part_plane_off", "part_planes", "part_bounds", "vis_vert_off",
               "vis_verts", "vis_tri_off", "vis_tris", "group_of_link")

    def __init__(self, fixture, urdf_path=None):
        """fixture: a prepared .hand.npz path, or the same arrays as a dict
        (e.g. oracle.ref_py.load_hand_arrays(urdf) for an ad-hoc URDF)."""
        z = np.load(fixture) if isinstance(fixture, (str, os.PathLike)) else fixture
        self.fixture = fixture if isinstance(fixture, (str, os.PathLike)) else None
        self.urdf = urdf_path
        self.arrays = {}
        for k in self._ARRAYS:
            dt = np.int32 if z[k].dtype.kind in "iu" else np.float64
            self.arrays[k] = np.ascontiguousarray(z[k], dtype=dt)
        self.link_names = [str(x) for x in z["link_names"]]
        self.joint_names = [str(x) for x in z["joint_names"]]
        self.n_groups = int(z["n_groups"])
        a = self.arrays
        d = A.HandDesc()
        d.n_links, d.dof, d.root = int(z["n_links"]), int(z["dof"]), int(z["root"])
        for f in ("parent", "joint_type", "joint_index", "topo_order", "part_link", "part_vert_off",
                  "part_tri_off", "part_tris", "part_plane_off"):
            setattr(d, f, _ip(a[f]))
        for f in ("origin_R", "origin_t", "axis", "limit_lo", "limit_hi", "part_verts",
                  "part_planes", "part_bounds"):
            setattr(d, f, _dp(a[f]))
        d.n_parts = len(a["part_link"])
        self.desc = d
        v = VisualDesc()
        v.n_links = d.n_links
        v.vert_off, v.verts = _ip(a["vis_vert_off"]), _dp(a["vis_verts"])
        v.tri_off, v.tris = _ip(a["vis_tri_off"]), _ip(a["vis_tris"])
        self.visual_desc = v
        self._names_c = (C.c_char_p * d.n_links)(*[s.encode() for s in self.joint_names])

    @property
    def n_links(self):
        return self.desc.n_links

    @property
    def dof(self):
        return self.desc.dof

    def link_name(self, l):
        return self.link_names[l]

    def groups(self):
        """dependency_groups (hand.cpp:374-411): (group id per link, n_groups)."""
        return self.arrays["group_of_link"].copy(), self.n_groups

    def link_visual(self, l):
        a = self.arrays
        v0, v1 = a["vis_vert_off"][l], a["vis_vert_off"][l + 1]
        t0, t1 = a["vis_tri_off"][l], a["vis_tri_off"][l + 1]
        return (a["vis_verts"].reshape(-1, 3)[v0:v1].copy(),
                a["vis_tris"].reshape(-1, 3)[t0:t1].copy())

    def limits(self):
        a = self.arrays
        lo, hi = np.zeros(self.dof), np.zeros(self.dof)
        for l in range(self.n_links):
            j = a["joint_index"][l]
            if j >= 0:
                lo[j], hi[j] = a["limit_lo"][l], a["limit_hi"][l]
        return lo, hi

    def mid_config(self):
        lo, hi = self.limits()
        return 0.5 * (lo + hi)


def load_hand(path, scale=1.0):
    """The reference's load_hand(path) result, from assets/prepared/."""
    if scale != 1.0:
        raise ValueError("prepared hand fixtures are at hand_scale 1.0")
    stem = os.path.splitext(os.path.basename(str(path)))[0]
    fx = os.path.join(PREPARED, f"{stem}.hand.npz")
    if not os.path.exists(fx):
        raise FileNotFoundError(f"{fx} missing: run tools/prepare_hands.py where the reference exists")
    return HandModel(fx, str(path))


class Patches:
    """decompose_patches output (contact_field.hpp:20-36) as lg_patches_desc,
    from the caller library (host) or the device (lg_hand_patches_device)."""

    def __init__(self, handle, destroy, export):
        self._h, self._destroy = handle, destroy
        self.desc = A.PatchesDesc()
        check(export(self._h, C.byref(self.desc)))

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                self._destroy(self._h)
            except Exception:
                pass
            self._h = None

    @property
    def n_patches(self):
        return self.desc.n_patches

    def link_of_patch(self):
        return np.ctypeslib.as_array(self.desc.link, shape=(self.n_patches,)).copy()


def hand_patches(hand, samples_per_cm2, patch_radius, seed, field_cap=8):
    """build_field's hand steps (pipeline.cpp:277-285) on the host: per-link
    samples with stream 'hnds' then decompose_patches (contact_field.cpp:26-99)."""
    h = C.c_void_p()
    check(lib().lgc_hand_patches(C.byref(hand.desc), C.byref(hand.visual_desc),
                                 float(samples_per_cm2), float(patch_radius), C.c_uint64(seed),
                                 int(field_cap), C.byref(h)))
    return Patches(h, lib().lgc_patches_destroy, lib().lgc_patches_export)


# ------------------------------------------------------------------ config
def default_config():
    p = A.RunParams()
    lib().lgc_run_params_default(C.byref(p))
    return p


def parse_config(path=None, hand=None, object=None, out=None, seed=None, batch=None,
                 workers=None):
    """parse_config (config.cpp:339-401) with CLI-style overrides."""
    p = A.RunParams()
    enc = (lambda s: None if s is None else str(s).encode())
    sd = None if seed is None else C.byref(C.c_longlong(int(seed)))
    bt = None if batch is None else C.byref(C.c_int(int(batch)))
    wk = None if workers is None else C.byref(C.c_int(int(workers)))
    check(lib().lgc_config_parse(enc(path), enc(hand), enc(object), enc(out), sd, bt, wk,
                                 C.byref(p)))
    return p


def index_cache_key(params):
    k = C.c_uint64()
    check(lib().lgc_index_cache_key(C.byref(params), C.byref(k)))
    return k.value


def write_dataset(path, grasps):
    """write_dataset (dataset.cpp:50-56): JSONL in the reference format."""
    g = np.ascontiguousarray(grasps)
    check(lib().lgc_write_dataset(str(path).encode(), g.ctypes.data_as(C.POINTER(A.Grasp)), len(g)))


def write_profile(path, profile_struct):
    check(lib().lgc_write_profile(str(path).encode(), C.byref(profile_struct)))


TAG_OBJECT_SAMPLES = 0x6F626A73  # pipeline.cpp:19


def prepare_object(params):
    """run_batch's object steps (pipeline.cpp:319-328): load, scale, sample."""
    mesh = load_mesh(params.object.decode())
    if params.object_scale != 1.0:
        mesh.scale(params.object_scale)
    raw = sample_surface(mesh, params.samples_per_cm2, mix_seed(params.seed, TAG_OBJECT_SAMPLES))
    return mesh, raw


def prepare_inputs(params):
    """Caller-side steps of run_batch / build_field (pipeline.cpp:273-330) on
    the host: the hand (prepared fixture), its patches, the object samples."""
    hand = load_hand(params.hand.decode(), params.hand_scale)
    patches = hand_patches(hand, params.samples_per_cm2, params.patch_radius, params.seed,
                           params.field_points_per_patch)
    mesh, raw = prepare_object(params)
    return hand, patches, raw, mesh
