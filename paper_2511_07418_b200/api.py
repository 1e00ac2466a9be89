"""Python mirror of the reference's C++ API over the lg.h C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/graspgen/*.hpp): load_hand, load_mesh,
sample_surface, decompose_patches (via hand_patches), parse_config,
ContactFieldIndex.build, query_domains, preprocess_object, run_batch,
write_dataset.  Exceptions map the C status codes back to the reference's
exception classes: invalid_argument -> ValueError, runtime_error ->
RuntimeError, out_of_range -> IndexError.

Every compute entry point runs on the GPU through libgraspgen_b200.so; there
is no CPU fallback, and a missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import lgabi as A

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgraspgen_b200.so")
_LIB = None


class CudaError(RuntimeError):
    """No CUDA device or a CUDA runtime failure (LG_ERR_CUDA)."""


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    P = C.POINTER
    sig = {
        "lg_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
        "lg_version": (C.c_char_p, []),
        "lg_index_cache_key": (C.c_int, [P(A.RunParams), P(C.c_uint64)]),
        "lg_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
        "lg_patches_export": (C.c_int, [vp, P(A.PatchesDesc)]),
        "lg_patches_destroy": (None, [vp]),
        "lg_device_count": (C.c_int, [A.ip]),
        "lg_ctx_create": (C.c_int, [C.c_int, P(vp)]),
        "lg_ctx_destroy": (None, [vp]),
        "lg_field_build": (C.c_int, [vp, P(A.HandDesc), P(A.PatchesDesc), C.c_int, C.c_double,
                                     C.c_uint64, C.c_int, P(vp)]),
        "lg_field_export": (C.c_int, [vp, P(A.FieldCsr)]),
        "lg_field_save": (C.c_int, [vp, C.c_char_p, C.c_uint64]),
        "lg_field_load": (C.c_int, [vp, P(A.HandDesc), C.c_char_p, C.c_uint64, P(vp)]),
        "lg_field_destroy": (None, [vp]),
        "lg_hand_patches_device": (C.c_int, [vp, P(A.HandDesc), vp, C.c_double, C.c_double,
                                             C.c_uint64, C.c_int, P(vp)]),
        "lg_patches_export": (C.c_int, [vp, P(A.PatchesDesc)]),
        "lg_patches_destroy": (None, [vp]),
        "lg_index_cache_key": (C.c_int, [P(A.RunParams), P(C.c_uint64)]),
        "lg_validate_batch": (C.c_int, [vp, P(A.HandDesc), vp, C.c_longlong, A.dp, C.c_int, A.ip,
                                        C.c_int, A.dp, C.c_int, P(A.RunParams), vp]),
        "lg_validation_issues": (C.c_int, [P(C.c_char_p), C.c_int, vp, C.c_longlong,
                                           P(A.RunParams), C.c_char_p, C.c_size_t, P(C.c_size_t),
                                           P(C.c_longlong)]),
        "lg_query_domains_batch": (C.c_int, [vp, vp, A.ip, A.dp, C.c_int, A.dp, C.c_int,
                                             C.c_double, P(C.c_uint32), A.dp]),
        "lg_preprocess": (C.c_int, [vp, A.dp, C.c_int, C.c_double, C.c_double,
                                    P(C.c_uint8)]),
        "lg_run_batch": (C.c_int, [vp, P(A.HandDesc), P(A.PatchesDesc), A.dp, C.c_int,
                                   P(A.RunParams), P(vp)]),
        "lg_run_batch_field": (C.c_int, [vp, P(A.HandDesc), P(A.PatchesDesc), vp, A.dp,
                                         C.c_int, P(A.RunParams), P(vp)]),
        "lg_result_profile": (C.c_int, [vp, P(A.Profile)]),
        "lg_result_num_grasps": (C.c_longlong, [vp]),
        "lg_result_grasps": (P(A.Grasp), [vp]),
        "lg_result_num_traces": (C.c_longlong, [vp]),
        "lg_result_traces": (P(A.Trace), [vp]),
        "lg_result_destroy": (None, [vp]),
        "lg_libm_eval": (C.c_int, [vp, C.c_int, C.c_longlong, A.dp, A.dp, A.dp]),
        "lg_debug_canary_violations": (C.c_longlong, []),
        "lg_query_domains_elements": (C.c_int, [vp, vp, A.ip, C.c_int, A.dp, C.c_int, A.dp,
                                                C.c_double, P(vp)]),
        "lg_domains_group": (C.c_int, [vp, C.c_int, P(C.c_longlong), P(C.c_longlong)]),
        "lg_domains_elements": (C.c_int, [vp, P(C.c_longlong), P(A.ip), P(A.dp), P(A.dp), P(A.dp),
                                          P(A.llp), P(A.ip), P(A.ip)]),
        "lg_domains_destroy": (None, [vp]),
        "lg_reverse_lookup_batch": (C.c_int, [vp, vp, C.c_int, A.llp, A.ip, A.ip, A.dp,
                                              P(C.c_uint64), A.ip, A.dp, A.dp]),
        "lg_place_batch": (C.c_int, [vp, P(A.HandDesc), P(A.PatchesDesc), vp, A.dp, C.c_int,
                                     P(A.RunParams), C.c_int, C.c_int, A.dp, A.ip, A.dp, A.ip,
                                     A.dp, A.dp, A.ip]),
        "lg_optimize_contacts_batch": (C.c_int, [vp, C.c_int, C.c_int, A.llp, A.dp, A.dp, A.ip,
                                                 A.dp, A.dp, P(A.RunParams), P(C.c_uint64), A.ip,
                                                 A.dp, A.ip, A.dp, A.dp, A.dp, A.llp]),
        "lg_realized_contacts_batch": (C.c_int, [vp, P(A.HandDesc), C.c_int, A.ip, A.dp, A.ip,
                                                 A.dp, A.dp, A.dp, A.ip, A.dp]),
        "lg_collision_report_batch": (C.c_int, [vp, P(A.HandDesc), C.c_int, A.dp, A.dp, A.dp,
                                                C.c_int, C.c_double, C.c_int, A.ip, A.ip, A.ip,
                                                A.dp, A.dp, A.ip]),
        "lg_comm_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
        "lg_comm_init": (C.c_int, [vp, C.POINTER(C.c_ubyte), C.c_int, C.c_int, P(vp)]),
        "lg_comm_destroy": (None, [vp]),
        "lg_comm_gather": (C.c_int, [vp, P(A.Grasp), C.c_longlong, P(A.Profile),
                                     P(P(A.Grasp)), P(C.c_longlong), P(A.Profile)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


def _err():
    buf = C.create_string_buffer(1024)
    lib().lg_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(rc):
    if rc == A.LG_OK:
        return
    msg = _err()
    if rc == A.LG_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == A.LG_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if rc == A.LG_ERR_CUDA:
        raise CudaError(msg)
    if rc == A.LG_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def _dp(a):
    return a.ctypes.data_as(A.dp)


def _ip(a):
    return a.ctypes.data_as(A.ip)


def mix_seed(seed, a, b=0):
    """mix_seed (rng.hpp:25-28)."""
    return int(lib().lg_mix_seed(C.c_uint64(seed), C.c_uint64(a), C.c_uint64(b)))


def index_cache_key(params):
    """index_cache_key (config.cpp:403-417), the GGCF cache key."""
    k = C.c_uint64()
    check(lib().lg_index_cache_key(C.byref(params), C.byref(k)))
    return k.value


class DevicePatches:
    """decompose_patches output built on the device (lg_hand_patches_device)."""

    def __init__(self, handle):
        self._h = handle
        self.desc = A.PatchesDesc()
        check(lib().lg_patches_export(self._h, C.byref(self.desc)))

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.lg_patches_destroy(self._h)
            self._h = None

    @property
    def n_patches(self):
        return self.desc.n_patches

    def link_of_patch(self):
        return np.ctypeslib.as_array(self.desc.link, shape=(self.n_patches,)).copy()


def hand_patches_device(ctx, hand, samples_per_cm2, patch_radius, seed, field_cap=8):
    """build_field's hand steps (pipeline.cpp:277-285) on the GPU: the
    per-link surface sampling, the greedy cover and the field-point subsets
    (identical patches).  `hand` carries .desc (lg_hand_desc) and
    .visual_desc (lg_visual_desc)."""
    h = C.c_void_p()
    check(lib().lg_hand_patches_device(ctx._h, C.byref(hand.desc), C.byref(hand.visual_desc),
                                       float(samples_per_cm2), float(patch_radius),
                                       C.c_uint64(seed), int(field_cap), C.byref(h)))
    return DevicePatches(h)


# ------------------------------------------------------------------ device
class Context:
    """One CUDA device + stream (one in-flight call per context)."""

    def __init__(self, device=0):
        h = C.c_void_p()
        check(lib().lg_ctx_create(int(device), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.lg_ctx_destroy(self._h)
            self._h = None

    __del__ = close


def device_count():
    n = C.c_int()
    check(lib().lg_device_count(C.byref(n)))
    return n.value


class ContactFieldIndex:
    """ContactFieldIndex (contact_field.hpp:112-137), resident on the GPU."""

    def __init__(self, handle, ctx):
        self._h = handle
        self._ctx = ctx

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.lg_field_destroy(self._h)
            self._h = None

    @classmethod
    def build(cls, ctx, hand, patches, N, box_width, seed, codebook_size=256):
        """ContactFieldIndex::build (contact_field.cpp:306-334) on the device."""
        h = C.c_void_p()
        check(lib().lg_field_build(ctx._h, C.byref(hand.desc), C.byref(patches.desc), int(N),
                                   float(box_width), C.c_uint64(seed), int(codebook_size),
                                   C.byref(h)))
        return cls(h, ctx)

    def save(self, path, key):
        """ContactFieldIndex::save (contact_field.cpp:570-600): GGCF v1 file."""
        check(lib().lg_field_save(self._h, os.fsencode(str(path)), C.c_uint64(key)))

    @classmethod
    def load(cls, ctx, hand, path, expected_key):
        """ContactFieldIndex::load (contact_field.cpp:602-655): None when the
        file is missing, malformed or keyed differently."""
        h = C.c_void_p()
        check(lib().lg_field_load(ctx._h, C.byref(hand.desc), os.fsencode(str(path)),
                                  C.c_uint64(expected_key), C.byref(h)))
        return cls(h, ctx) if h.value else None

    def export(self):
        """Host CSR copy: patches -> boxes (lexicographic cells) -> codes/reps."""
        o = A.FieldCsr()
        check(lib().lg_field_export(self._h, C.byref(o)))
        P, B, Q = o.n_patches, o.n_boxes, o.n_codes
        arr = np.ctypeslib.as_array
        return dict(
            box_width=o.box_width,
            codebook=arr(o.codebook, shape=(o.codebook_size * 3,)).reshape(-1, 3).copy(),
            patch_link=arr(o.patch_link, shape=(P,)).copy(),
            patch_box_off=arr(o.patch_box_off, shape=(P + 1,)).copy(),
            box_cell=arr(o.box_cell, shape=(B * 3,)).reshape(-1, 3).copy(),
            box_code_off=arr(o.box_code_off, shape=(B + 1,)).copy(),
            codes=arr(o.codes, shape=(Q,)).copy(),
            rep_link=arr(o.rep_link, shape=(Q,)).copy(),
            rep_point=arr(o.rep_point, shape=(Q * 3,)).reshape(-1, 3).copy(),
            rep_normal=arr(o.rep_normal, shape=(Q * 3,)).reshape(-1, 3).copy(),
            n_vectors=o.n_vectors,
        )


def query_domains_batch(ctx, field, group_of_patch, samples, poses, theta_hit,
                        with_scores=False):
    """query_domains (contact_field.cpp:380-448) for m poses: reachability
    masks (m, n) uint32, bit g = sample is an element of group g's domain;
    with_scores also returns the element scores (m, n) (max over the
    sample's elements, 0 without one)."""
    s = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 6)
    p = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 12)
    g = np.ascontiguousarray(group_of_patch, dtype=np.int32)
    masks = np.zeros((len(p), len(s)), dtype=np.uint32)
    scores = np.zeros((len(p), len(s))) if with_scores else None
    check(lib().lg_query_domains_batch(ctx._h, field._h, _ip(g), _dp(s), len(s), _dp(p), len(p),
                                       float(theta_hit),
                                       masks.ctypes.data_as(C.POINTER(C.c_uint32)),
                                       _dp(scores) if with_scores else None))
    return (masks, scores) if with_scores else masks


def libm_eval(ctx, which, x, y=None):
    """The device's sin/cos/log/atan2/hypot (glibc's algorithms, lg_libm.h)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    yy = np.ascontiguousarray(x if y is None else y, dtype=np.float64)
    out = np.zeros_like(x)
    idx = {"sin": 0, "cos": 1, "log": 2, "atan2": 3, "hypot": 4}[which]
    check(lib().lg_libm_eval(ctx._h, idx, len(x), _dp(x), _dp(yy), _dp(out)))
    return out


def preprocess_object(ctx, samples, probe_half_width, depth_threshold):
    """preprocess_object (pipeline.cpp:71-98) -> keep mask (bool, order kept)."""
    s = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 6)
    keep = np.zeros(len(s), dtype=np.uint8)
    check(lib().lg_preprocess(ctx._h, _dp(s), len(s), float(probe_half_width),
                              float(depth_threshold), keep.ctypes.data_as(C.POINTER(C.c_uint8))))
    return keep.astype(bool)


class RunResult:
    """RunResult (pipeline.hpp:143-148): grasps, StageProfile, traces."""

    def __init__(self, handle):
        L = lib()
        self.profile_struct = A.Profile()
        check(L.lg_result_profile(handle, C.byref(self.profile_struct)))
        self.profile = {n: getattr(self.profile_struct, n) for n, _ in A.Profile._fields_}
        ng = L.lg_result_num_grasps(handle)
        nt = L.lg_result_num_traces(handle)
        self.grasps = _copy_structs(L.lg_result_grasps(handle), ng, A.grasp_dtype())
        self.traces = _copy_structs(L.lg_result_traces(handle), nt, A.trace_dtype())
        L.lg_result_destroy(handle)


def _copy_structs(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (n * dtype.itemsize)).from_address(C.cast(ptr, C.c_void_p).value)
    return np.frombuffer(bytes(buf), dtype=dtype).copy()


def run_batch(ctx, hand, patches, raw_samples, params, field=None):
    """run_batch (pipeline.cpp:308-625) on the GPU: field build (unless a
    prebuilt field is given), preprocess, placement, domains, contact search,
    realisation and postprocess."""
    raw = np.ascontiguousarray(raw_samples, dtype=np.float64).reshape(-1, 6)
    h = C.c_void_p()
    if field is None:
        check(lib().lg_run_batch(ctx._h, C.byref(hand.desc), C.byref(patches.desc), _dp(raw),
                                 len(raw), C.byref(params), C.byref(h)))
    else:
        check(lib().lg_run_batch_field(ctx._h, C.byref(hand.desc), C.byref(patches.desc),
                                       field._h, _dp(raw), len(raw), C.byref(params),
                                       C.byref(h)))
    return RunResult(h)


def validate_batch(ctx, hand, grasps, mesh, samples, params):
    """validate_dataset (validate.cpp:56-175) on the GPU: per-grasp checks
    (structured array of lg_grasp_check)."""
    g = np.ascontiguousarray(np.asarray(grasps).astype(A.grasp_dtype()))
    v, t = mesh.arrays() if hasattr(mesh, "arrays") else mesh
    v = np.ascontiguousarray(v, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.int32)
    s = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 6)
    out = np.zeros(len(g), dtype=A.check_dtype())
    check(lib().lg_validate_batch(ctx._h, C.byref(hand.desc), g.ctypes.data_as(C.c_void_p), len(g),
                                  _dp(v), len(v), _ip(t), len(t), _dp(s), len(s), C.byref(params),
                                  out.ctypes.data_as(C.c_void_p)))
    return out


def validation_issues(joint_names, checks, params):
    """ValidationReport.issues as [(grasp, message)], texts as validate.cpp
    words them; joint_names = joint name per link (Link::joint_name)."""
    c = np.ascontiguousarray(checks)
    names = (C.c_char_p * max(1, len(joint_names)))(*[str(n).encode() for n in joint_names])
    need, cnt = C.c_size_t(0), C.c_longlong(0)
    check(lib().lg_validation_issues(names, len(joint_names), c.ctypes.data_as(C.c_void_p), len(c),
                                     C.byref(params), None, 0, C.byref(need), C.byref(cnt)))
    buf = C.create_string_buffer(need.value)
    check(lib().lg_validation_issues(names, len(joint_names), c.ctypes.data_as(C.c_void_p), len(c),
                                     C.byref(params), buf, need.value, C.byref(need),
                                     C.byref(cnt)))
    out = []
    for line in buf.value.decode().splitlines():
        gi, what = line.split("\t", 1)
        out.append((int(gi), what))
    return out


def _bind_batch_sigs():
    L = lib()
    if getattr(L, "_batch_bound", False):
        return L
    P = C.POINTER
    L.lg_wrench_solve_batch.restype = C.c_int
    L.lg_wrench_solve_batch.argtypes = [C.c_void_p, C.c_int, A.ip, A.dp, A.dp, C.c_double,
                                        C.c_double, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_int, A.dp, A.ip, A.dp, A.dp, A.dp]
    L.lg_collision_batch.restype = C.c_int
    L.lg_collision_batch.argtypes = [C.c_void_p, P(A.HandDesc), C.c_int, A.dp, A.dp, A.dp,
                                     C.c_int, C.c_double, P(C.c_uint8), A.dp]
    L.lg_realize_batch.restype = C.c_int
    L.lg_realize_batch.argtypes = [C.c_void_p, P(A.HandDesc), C.c_int, A.ip, A.dp, A.dp, A.ip,
                                   A.dp, A.dp, C.c_double, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_int, C.c_int, A.dp, A.dp, A.ip,
                                   P(C.c_ulonglong)]
    L.lg_contact_ik_batch.restype = C.c_int
    L.lg_contact_ik_batch.argtypes = [C.c_void_p, P(A.HandDesc), C.c_int, A.ip, A.dp, A.dp, A.dp,
                                      A.ip, A.dp, A.dp, C.c_double, C.c_int, C.c_double,
                                      C.c_double, C.c_double, C.c_double, C.c_int, A.dp, A.ip,
                                      P(C.c_ulonglong), A.ip, A.dp, A.dp, A.dp]
    L._batch_bound = True
    return L


def wrench_solve_batch(ctx, problems, lambda_torque=10.0, mu=0.0, gswo=None, iterations=64,
                       warm_iterations=8, step=0.1, max_backtracks=20):
    """Batched solve_fswo / solve_gswo (wrench.cpp:247-258), cold start.
    problems: list of (points (n,3), inward normals (n,3)), n <= 6."""
    L = _bind_batch_sigs()
    m = len(problems)
    n = np.array([len(p[0]) for p in problems], dtype=np.int32)
    if m and (n.min() < 1 or n.max() > 6):
        raise ValueError("wrench solve: 1..6 contacts")  # as the C-ABI reports it
    pts = np.zeros((m, 6, 3))
    nrm = np.zeros((m, 6, 3))
    for i, (p, q) in enumerate(problems):
        pts[i, :len(p)] = p
        nrm[i, :len(q)] = q
    mode = (1 if mu > 0 else 0) if gswo is None else int(gswo)
    obj = np.zeros(m)
    anchor = np.zeros(m, dtype=np.int32)
    al, bx, by = np.zeros((m, 6)), np.zeros((m, 6)), np.zeros((m, 6))
    check(L.lg_wrench_solve_batch(lib_ctx(ctx), m, _ip(n), _dp(pts), _dp(nrm),
                                  float(lambda_torque), float(mu), mode, int(iterations),
                                  int(warm_iterations), float(step), int(max_backtracks),
                                  _dp(obj), _ip(anchor), _dp(al), _dp(bx), _dp(by)))
    return obj, anchor, al, bx, by


def lib_ctx(ctx):
    return ctx._h


def collision_batch(ctx, hand, q, poses, samples, margin=0.002):
    """Batched validate_grasp_collisions (collision.cpp:230-288) -> (clean, max depth)."""
    L = _bind_batch_sigs()
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, hand.dof)
    p = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 12)
    s = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 6)
    m = len(q)
    clean = np.zeros(m, dtype=np.uint8)
    mp = np.zeros(m)
    check(L.lg_collision_batch(ctx._h, C.byref(hand.desc), m, _dp(q), _dp(p), _dp(s), len(s),
                               float(margin), clean.ctypes.data_as(C.POINTER(C.c_uint8)), _dp(mp)))
    return clean.astype(bool), mp


def contact_ik_batch(ctx, hand, q0, problems, beta=0.01, iterations=30, step_clamp=0.2,
                     residual_tol=1e-4, damping_scale=1e-4, damping_min=1e-6, max_backtracks=10):
    """Batched solve_contact_ik (ik.cpp:30-139).  problems: list of target
    lists, each target (object_point, inward normal, link, hand point, hand
    normal).  Returns a dict of q, finite, used_joints, iterations, objective,
    and per problem the position residuals and clamped normal cosines."""
    L = _bind_batch_sigs()
    m = len(problems)
    k = np.array([len(t) for t in problems], dtype=np.int32)
    flat = [t for ts in problems for t in ts]
    nt = max(len(flat), 1)
    op = np.ascontiguousarray([t[0] for t in flat] or [[0, 0, 0]], dtype=np.float64).reshape(-1, 3)
    on = np.ascontiguousarray([t[1] for t in flat] or [[0, 0, 0]], dtype=np.float64).reshape(-1, 3)
    links = np.ascontiguousarray([t[2] for t in flat] or [0], dtype=np.int32)
    hp = np.ascontiguousarray([t[3] for t in flat] or [[0, 0, 0]], dtype=np.float64).reshape(-1, 3)
    hn = np.ascontiguousarray([t[4] for t in flat] or [[0, 0, 0]], dtype=np.float64).reshape(-1, 3)
    q0 = np.ascontiguousarray(q0, dtype=np.float64).reshape(m, hand.dof)
    q = np.zeros_like(q0)
    fin = np.zeros(m, dtype=np.int32)
    used = np.zeros(m, dtype=np.uint64)
    its = np.zeros(m, dtype=np.int32)
    obj = np.zeros(m)
    pos, cos = np.zeros(nt), np.zeros(nt)
    check(L.lg_contact_ik_batch(ctx._h, C.byref(hand.desc), m, _ip(k), _dp(q0), _dp(op), _dp(on),
                                _ip(links), _dp(hp), _dp(hn), beta, iterations, step_clamp,
                                residual_tol, damping_scale, damping_min, max_backtracks, _dp(q),
                                _ip(fin), used.ctypes.data_as(C.POINTER(C.c_ulonglong)), _ip(its),
                                _dp(obj), _dp(pos), _dp(cos)))
    off = np.concatenate([[0], np.cumsum(k)])
    return {"q": q, "finite": fin, "used_joints": used, "iterations": its, "objective": obj,
            "position": [pos[off[i]:off[i + 1]] for i in range(m)],
            "cosine": [cos[off[i]:off[i + 1]] for i in range(m)]}


def realize_batch(ctx, hand, q0, problems, beta=0.01, iterations=30, step_clamp=0.2,
                  residual_tol=1e-4, damping_scale=1e-4, finetune_rounds=4,
                  finetune_iterations=10):
    """Batched realize_grasp (pipeline.cpp:185-253).  problems: list of target
    lists, each target (object_point, inward normal, link, hand point, hand normal)."""
    L = _bind_batch_sigs()
    m = len(problems)
    k = np.array([len(t) for t in problems], dtype=np.int32)
    flat = [t for ts in problems for t in ts]
    op = np.ascontiguousarray([t[0] for t in flat], dtype=np.float64).reshape(-1, 3)
    on = np.ascontiguousarray([t[1] for t in flat], dtype=np.float64).reshape(-1, 3)
    links = np.ascontiguousarray([t[2] for t in flat], dtype=np.int32)
    hp = np.ascontiguousarray([t[3] for t in flat], dtype=np.float64).reshape(-1, 3)
    hn = np.ascontiguousarray([t[4] for t in flat], dtype=np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(np.broadcast_to(q0, (m, hand.dof)), dtype=np.float64).copy()
    mr = np.zeros(m)
    fin = np.zeros(m, dtype=np.int32)
    used = np.zeros(m, dtype=np.uint64)
    check(L.lg_realize_batch(ctx._h, C.byref(hand.desc), m, _ip(k), _dp(op), _dp(on), _ip(links),
                             _dp(hp), _dp(hn), float(beta), int(iterations), float(step_clamp),
                             float(residual_tol), float(damping_scale), int(finetune_rounds),
                             int(finetune_iterations), _dp(q), _dp(mr), _ip(fin),
                             used.ctypes.data_as(C.POINTER(C.c_ulonglong))))
    return q, mr, fin.astype(bool), used


# ------------------------------------------------ stage-level entry points
def _llp(a):
    return a.ctypes.data_as(A.llp)


def query_domains_elements(ctx, field, group_of_patch, n_groups, samples, pose12, theta_hit):
    """query_domains (contact_field.cpp:380-448) for one pose: list over
    groups of element dicts {sample, pos, nrm, score, hits: [(patch, box)]}."""
    s = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 6)
    g = np.ascontiguousarray(group_of_patch, dtype=np.int32)
    pose = np.ascontiguousarray(pose12, dtype=np.float64).reshape(12)
    L = lib()
    h = C.c_void_p()
    check(L.lg_query_domains_elements(ctx._h, field._h, _ip(g), int(n_groups), _dp(s), len(s),
                                      _dp(pose), float(theta_hit), C.byref(h)))
    try:
        n = C.c_longlong(0)
        sp, pp, nn, sc, ho, hp, hb = (A.ip(), A.dp(), A.dp(), A.dp(), A.llp(), A.ip(), A.ip())
        check(L.lg_domains_elements(h, C.byref(n), C.byref(sp), C.byref(pp), C.byref(nn),
                                    C.byref(sc), C.byref(ho), C.byref(hp), C.byref(hb)))
        E = n.value
        arr = np.ctypeslib.as_array
        off = arr(ho, shape=(E + 1,)).copy() if E else np.zeros(1, np.int64)
        H = int(off[-1])
        sample = arr(sp, shape=(E,)).copy() if E else np.zeros(0, np.int32)
        pos = arr(pp, shape=(3 * E,)).reshape(-1, 3).copy() if E else np.zeros((0, 3))
        nrm = arr(nn, shape=(3 * E,)).reshape(-1, 3).copy() if E else np.zeros((0, 3))
        score = arr(sc, shape=(E,)).copy() if E else np.zeros(0)
        hpa = arr(hp, shape=(H,)).copy() if H else np.zeros(0, np.int32)
        hba = arr(hb, shape=(H,)).copy() if H else np.zeros(0, np.int32)
        out = []
        for grp in range(int(n_groups)):
            f, c = C.c_longlong(0), C.c_longlong(0)
            check(L.lg_domains_group(h, grp, C.byref(f), C.byref(c)))
            els = []
            for e in range(f.value, f.value + c.value):
                els.append({"sample": int(sample[e]), "pos": pos[e], "nrm": nrm[e],
                            "score": float(score[e]),
                            "hits": list(zip(hpa[off[e]:off[e + 1]].tolist(),
                                             hba[off[e]:off[e + 1]].tolist()))})
            out.append(els)
        return out
    finally:
        L.lg_domains_destroy(h)


def reverse_lookup_batch(ctx, field, elements, seeds):
    """reverse_lookup (contact_field.cpp:450-484) for elements (dicts with
    'hits' and 'nrm') -> (links, points, normals)."""
    m = len(elements)
    off = np.zeros(m + 1, dtype=np.int64)
    for i, e in enumerate(elements):
        off[i + 1] = off[i] + len(e["hits"])
    hp = np.array([h[0] for e in elements for h in e["hits"]] or [0], dtype=np.int32)
    hb = np.array([h[1] for e in elements for h in e["hits"]] or [0], dtype=np.int32)
    nr = np.ascontiguousarray([e["nrm"] for e in elements], dtype=np.float64).reshape(-1, 3)
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    link = np.zeros(m, dtype=np.int32)
    pt, nn = np.zeros((m, 3)), np.zeros((m, 3))
    check(lib().lg_reverse_lookup_batch(ctx._h, field._h, m, _llp(off), _ip(hp), _ip(hb), _dp(nr),
                                        sd.ctypes.data_as(C.POINTER(C.c_uint64)), _ip(link),
                                        _dp(pt), _dp(nn)))
    return link, pt, nn


def place_batch(ctx, hand, patches, raw_samples, params, c0, m, field=None):
    """place_object (pipeline.cpp:122-183) for candidates [c0, c0+m)."""
    raw = np.ascontiguousarray(raw_samples, dtype=np.float64).reshape(-1, 6)
    pose = np.zeros((m, 12))
    acc, nst, stl = (np.zeros(m, np.int32) for _ in range(3))
    pen = np.zeros(m)
    stp, stn = np.zeros((m, 3)), np.zeros((m, 3))
    check(lib().lg_place_batch(ctx._h, C.byref(hand.desc), C.byref(patches.desc),
                               field._h if field is not None else None, _dp(raw), len(raw),
                               C.byref(params), int(c0), int(m), _dp(pose), _ip(acc), _dp(pen),
                               _ip(nst), _dp(stp), _dp(stn), _ip(stl)))
    return dict(pose=pose, accepted=acc, penetration=pen, n_static=nst, static_p=stp,
                static_n=stn, static_link=stl)


def optimize_contacts_batch(ctx, problems, params, seeds):
    """optimize_contacts (contact_opt.cpp:45-142); problems = [(domains,
    statics)] with domains = [(positions [n,3], normals [n,3])] * k and
    statics = [] or [(p, n)]."""
    m = len(problems)
    k = len(problems[0][0])
    off = [0]
    P, N = [], []
    nst = np.zeros(m, np.int32)
    sp, sn = np.zeros((m, 3)), np.zeros((m, 3))
    for i, (doms, st) in enumerate(problems):
        assert len(doms) == k
        for pos, nrm in doms:
            pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
            P.append(pos)
            N.append(np.asarray(nrm, dtype=np.float64).reshape(-1, 3))
            off.append(off[-1] + len(pos))
        if st:
            nst[i] = 1
            sp[i], sn[i] = st[0][0], st[0][1]
    off = np.array(off, dtype=np.int64)
    P = np.ascontiguousarray(np.concatenate(P))
    N = np.ascontiguousarray(np.concatenate(N))
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    ids = np.zeros((m, k), np.int32)
    obj = np.zeros(m)
    anc = np.zeros(m, np.int32)
    al, bx, by = np.zeros((m, 6)), np.zeros((m, 6)), np.zeros((m, 6))
    ev = np.zeros(m, np.int64)
    check(lib().lg_optimize_contacts_batch(ctx._h, m, k, _llp(off), _dp(P), _dp(N), _ip(nst), _dp(sp),
                                           _dp(sn), C.byref(params),
                                           sd.ctypes.data_as(C.POINTER(C.c_uint64)), _ip(ids),
                                           _dp(obj), _ip(anc), _dp(al), _dp(bx), _dp(by),
                                           _llp(ev)))
    return dict(element_ids=ids, objective=obj, anchor=anc, alpha=al, beta_x=bx, beta_y=by,
                evaluations=ev)


def realized_contacts_batch(ctx, hand, q, problems):
    """realize_grasp's final projection: problems = [[(link, object_point)]]."""
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(len(problems), -1)
    k = np.array([len(t) for t in problems], np.int32)
    links = np.array([l for t in problems for l, _ in t], np.int32)
    op = np.ascontiguousarray([p for t in problems for _, p in t], dtype=np.float64).reshape(-1, 3)
    n = len(links)
    rp, rn, rs = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n)
    rl = np.zeros(n, np.int32)
    check(lib().lg_realized_contacts_batch(ctx._h, C.byref(hand.desc), len(problems), _ip(k), _dp(q),
                                           _ip(links), _dp(op), _dp(rp), _dp(rn), _ip(rl), _dp(rs)))
    return rp, rn, rl, rs


def collision_report_batch(ctx, hand, q, poses, samples, margin=0.002, cap=64):
    """validate_grasp_collisions' CollisionReport for each configuration."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    m = q.shape[0]
    poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(m, 12)
    s = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 6)
    nv, bp = np.zeros(m, np.int32), np.zeros((m, 3), np.int32)
    la, lb = np.zeros((m, cap), np.int32), np.zeros((m, cap), np.int32)
    dd, mp = np.zeros((m, cap)), np.zeros(m)
    check(lib().lg_collision_report_batch(ctx._h, C.byref(hand.desc), m, _dp(q), _dp(poses), _dp(s),
                                          len(s), float(margin), int(cap), _ip(nv), _ip(la),
                                          _ip(lb), _dp(dd), _dp(mp), _ip(bp)))
    out = []
    for i in range(m):
        n = min(nv[i], cap)
        out.append(dict(n_violations=int(nv[i]), max_penetration=float(mp[i]),
                        broad_pairs=int(bp[i, 0]), narrow_gjk=int(bp[i, 1]),
                        narrow_halfplane=int(bp[i, 2]),
                        violations=list(zip(la[i, :n].tolist(), lb[i, :n].tolist(),
                                            dd[i, :n].tolist()))))
    return out
