"""ctypes binding of the CPU parity oracle (oracle/liborc.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2511_07418_b200 import lgabi as A

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ORC_LIB", os.path.join(_HERE, "liborc.so"))
_LIB = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, P, dp, ip = C.c_void_p, C.POINTER, A.dp, A.ip
        HD, PD = P(A.HandDesc), P(A.PatchesDesc)
        sig = {
            "orc_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
            "orc_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
            "orc_rng_u64": (None, [C.c_uint64, C.c_int, P(C.c_uint64)]),
            "orc_rng_normal": (None, [C.c_uint64, C.c_int, dp]),
            "orc_rng_unit_vectors": (None, [C.c_uint64, C.c_int, dp]),
            "orc_rng_quaternions": (None, [C.c_uint64, C.c_int, dp]),
            "orc_libm": (None, [C.c_int, C.c_int, dp, dp, dp]),
            "orc_glibc": (None, [C.c_int, C.c_longlong, dp, dp, dp]),
            "orc_tangent_basis": (C.c_int, [dp, dp, dp]),
            "orc_rotation_between": (C.c_int, [dp, dp, dp]),
            "orc_fk": (C.c_int, [HD, dp, dp]),
            "orc_point_jacobian": (C.c_int, [HD, dp, C.c_int, dp, dp]),
            "orc_groups": (C.c_int, [HD, ip, ip]),
            "orc_sample_surface": (C.c_int, [dp, C.c_int, ip, C.c_int, C.c_double, C.c_uint64,
                                             dp, C.c_size_t, P(C.c_size_t)]),
            "orc_decompose_patches": (C.c_int, [HD, dp, ip, C.c_double, C.c_uint64, C.c_int,
                                                P(vp)]),
            "orc_patches_export": (C.c_int, [vp, PD]),
            "orc_patches_destroy": (None, [vp]),
            "orc_field_build": (C.c_int, [HD, PD, C.c_int, C.c_double, C.c_uint64, C.c_int,
                                          P(vp)]),
            "orc_field_export": (C.c_int, [vp, P(A.FieldCsr)]),
            "orc_field_nodes": (C.c_longlong, [vp]),
            "orc_field_save": (C.c_int, [vp, C.c_char_p, C.c_uint64]),
            "orc_validate": (C.c_int, [HD, vp, C.c_longlong, dp, C.c_int, ip, C.c_int, dp, C.c_int,
                                       P(A.RunParams), vp]),
            "orc_field_destroy": (None, [vp]),
            "orc_query": (C.c_int, [vp, HD, dp, C.c_int, dp, C.c_double, P(C.c_uint32), dp, ip]),
            "orc_reverse_lookup": (C.c_int, [vp, HD, dp, C.c_int, dp, C.c_double, C.c_int,
                                             C.c_int, C.c_uint64, ip, dp, dp]),
            "orc_preprocess": (C.c_int, [dp, C.c_int, C.c_double, C.c_double, P(C.c_uint8)]),
            "orc_wrench_solve": (C.c_int, [C.c_int, dp, dp, C.c_double, C.c_double, C.c_int,
                                           C.c_int, C.c_int, C.c_double, C.c_int, dp, dp, dp,
                                           dp, ip, dp, dp, dp]),
            "orc_wrench_objective": (C.c_int, [C.c_int, dp, dp, C.c_double, C.c_double, dp, dp,
                                               dp, dp]),
            "orc_optimize_contacts": (C.c_int, [C.c_int, ip, dp, dp, C.c_int, dp, dp, C.c_int,
                                                C.c_int, C.c_int, C.c_double, C.c_double,
                                                C.c_double, C.c_uint64, ip, dp, ip]),
            "orc_collision": (C.c_int, [HD, dp, dp, dp, C.c_int, C.c_double, ip, dp, ip]),
            "orc_gjk": (C.c_int, [HD, C.c_int, dp, C.c_int, dp, dp]),
            "orc_closest_on_parts": (C.c_int, [HD, C.c_int, dp, dp, dp, dp]),
            "orc_ik": (C.c_int, [HD, dp, C.c_int, dp, dp, ip, dp, dp, C.c_double, C.c_int,
                                 C.c_double, C.c_double, C.c_double, dp, ip, dp, ip,
                                 P(C.c_ulonglong), dp, dp]),
            "orc_realize": (C.c_int, [HD, dp, C.c_int, dp, dp, ip, dp, dp, C.c_double, C.c_int,
                                      C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, dp,
                                      dp, ip, P(C.c_ulonglong)]),
            "orc_run_batch": (C.c_int, [HD, PD, dp, C.c_int, P(A.RunParams), C.c_int, P(vp)]),
            "orc_run_batch_field": (C.c_int, [vp, HD, PD, dp, C.c_int, P(A.RunParams), C.c_int,
                                              P(vp)]),
            "orc_result_profile": (C.c_int, [vp, P(A.Profile)]),
            "orc_result_num_grasps": (C.c_longlong, [vp]),
            "orc_result_grasps": (P(A.Grasp), [vp]),
            "orc_result_num_traces": (C.c_longlong, [vp]),
            "orc_result_traces": (P(A.Trace), [vp]),
            "orc_result_destroy": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc):
    if rc == 0:
        return
    buf = C.create_string_buffer(1024)
    lib().orc_last_error(buf, 1024)
    msg = buf.value.decode(errors="replace")
    if rc == A.LG_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == A.LG_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(A.dp)


def _i(a):
    return a.ctypes.data_as(A.ip)


def rng_u64(seed, n):
    out = np.zeros(n, dtype=np.uint64)
    lib().orc_rng_u64(C.c_uint64(seed), n, out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def rng_normal(seed, n):
    out = np.zeros(n)
    lib().orc_rng_normal(C.c_uint64(seed), n, _p(out))
    return out


def rng_unit_vectors(seed, n):
    out = np.zeros((n, 3))
    lib().orc_rng_unit_vectors(C.c_uint64(seed), n, _p(out))
    return out


def rng_quaternions(seed, n):
    out = np.zeros((n, 4))
    lib().orc_rng_quaternions(C.c_uint64(seed), n, _p(out))
    return out


def libm(which, x, y=None):
    x = _d(x)
    y = _d(x if y is None else y)
    out = np.zeros_like(x)
    idx = {"sin": 0, "cos": 1, "log": 2, "atan2": 3, "hypot": 4}[which]
    lib().orc_libm(idx, len(x), _p(x), _p(y), _p(out))
    return out


def glibc(which, x, y=None):
    """The host glibc's own std::sin/cos/log/atan2/hypot (what the reference
    calls), evaluated natively over the arrays."""
    x = _d(x)
    y = _d(x if y is None else y)
    out = np.zeros_like(x)
    idx = {"sin": 0, "cos": 1, "log": 2, "atan2": 3, "hypot": 4}[which]
    lib().orc_glibc(idx, len(x), _p(x), _p(y), _p(out))
    return out


def hypot_exceeds(x, y, cap):
    x, y, cap = _d(x), _d(y), _d(cap)
    out = np.zeros(len(x), dtype=np.uint8)
    lib().orc_hypot_exceeds(C.c_longlong(len(x)), _p(x), _p(y), _p(cap),
                            out.ctypes.data_as(C.POINTER(C.c_uint8)))
    return out.astype(bool)


def mix_seed(s, a, b=0):
    return int(lib().orc_mix_seed(C.c_uint64(s), C.c_uint64(a), C.c_uint64(b)))


def tangent_basis(n):
    n = _d(n)
    x, y = np.zeros(3), np.zeros(3)
    check(lib().orc_tangent_basis(_p(n), _p(x), _p(y)))
    return x, y


def rotation_between(a, b):
    a, b = _d(a), _d(b)
    R = np.zeros(9)
    check(lib().orc_rotation_between(_p(a), _p(b), _p(R)))
    return R.reshape(3, 3)


def fk(hand_desc, q):
    q = _d(q)
    out = np.zeros(hand_desc.n_links * 12)
    check(lib().orc_fk(C.byref(hand_desc), _p(q), _p(out)))
    return out.reshape(-1, 12)


def point_jacobian(hand_desc, q, link, local_point):
    q, lp = _d(q), _d(local_point)
    J = np.zeros(3 * hand_desc.dof)
    check(lib().orc_point_jacobian(C.byref(hand_desc), _p(q), int(link), _p(lp), _p(J)))
    return J.reshape(3, -1)


def groups(hand_desc):
    g = np.zeros(hand_desc.n_links, dtype=np.int32)
    n = C.c_int()
    check(lib().orc_groups(C.byref(hand_desc), _i(g), C.byref(n)))
    return g, n.value


def sample_surface(verts, tris, spc, seed):
    v = _d(verts).reshape(-1, 3)
    t = np.ascontiguousarray(tris, dtype=np.int32).reshape(-1, 3)
    n = C.c_size_t()
    check(lib().orc_sample_surface(_p(v), len(v), _i(t), len(t), float(spc), C.c_uint64(seed),
                                   None, 0, C.byref(n)))
    out = np.zeros((n.value, 6))
    check(lib().orc_sample_surface(_p(v), len(v), _i(t), len(t), float(spc), C.c_uint64(seed),
                                   _p(out), n.value, C.byref(n)))
    return out


class OrcPatches:
    def __init__(self, hand_desc, per_link_samples, radius, seed, cap=8):
        off = np.zeros(len(per_link_samples) + 1, dtype=np.int32)
        for i, s in enumerate(per_link_samples):
            off[i + 1] = off[i] + len(s)
        cat = _d(np.concatenate([np.asarray(s).reshape(-1, 6) for s in per_link_samples]))
        h = C.c_void_p()
        check(lib().orc_decompose_patches(C.byref(hand_desc), _p(cat), _i(off), float(radius),
                                          C.c_uint64(seed), int(cap), C.byref(h)))
        self._h = h
        self.desc = A.PatchesDesc()
        lib().orc_patches_export(self._h, C.byref(self.desc))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_patches_destroy(self._h)
            self._h = None


class OrcField:
    def __init__(self, hand_desc, patches_desc, N, w, seed, C_=256):
        h = C.c_void_p()
        check(lib().orc_field_build(C.byref(hand_desc), C.byref(patches_desc), int(N), float(w),
                                    C.c_uint64(seed), int(C_), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_field_destroy(self._h)
            self._h = None

    def export(self):
        o = A.FieldCsr()
        lib().orc_field_export(self._h, C.byref(o))
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

    def nodes(self):
        return int(lib().orc_field_nodes(self._h))

    def save(self, path, key):
        """ContactFieldIndex::save (contact_field.cpp:570-600)."""
        check(lib().orc_field_save(self._h, str(path).encode(), C.c_uint64(key)))

    def query(self, hand_desc, samples, pose12, theta):
        s = _d(samples).reshape(-1, 6)
        p = _d(pose12)
        masks = np.zeros(len(s), dtype=np.uint32)
        scores = np.zeros(len(s))
        sizes = np.zeros(32, dtype=np.int32)
        check(lib().orc_query(self._h, C.byref(hand_desc), _p(s), len(s), _p(p), float(theta),
                              masks.ctypes.data_as(C.POINTER(C.c_uint32)), _p(scores), _i(sizes)))
        return masks, scores, sizes

    def reverse_lookup(self, hand_desc, samples, pose12, theta, sample, group, seed):
        s = _d(samples).reshape(-1, 6)
        p = _d(pose12)
        link = C.c_int()
        pt, nr = np.zeros(3), np.zeros(3)
        check(lib().orc_reverse_lookup(self._h, C.byref(hand_desc), _p(s), len(s), _p(p),
                                       float(theta), int(sample), int(group), C.c_uint64(seed),
                                       C.byref(link), _p(pt), _p(nr)))
        return link.value, pt, nr


def preprocess(samples, h, d):
    s = _d(samples).reshape(-1, 6)
    keep = np.zeros(len(s), dtype=np.uint8)
    check(lib().orc_preprocess(_p(s), len(s), float(h), float(d),
                               keep.ctypes.data_as(C.POINTER(C.c_uint8))))
    return keep.astype(bool)


def wrench_solve(points, normals, lam=10.0, mu=0.0, mode=None, iterations=64, warm_iterations=8,
                 step=0.1, max_backtracks=20, warm=None):
    p, n = _d(points).reshape(-1, 3), _d(normals).reshape(-1, 3)
    k = len(p)
    mode = (1 if mu > 0 else 0) if mode is None else mode
    obj = C.c_double()
    anchor = C.c_int()
    al, bx, by = np.zeros(k), np.zeros(k), np.zeros(k)
    wa = wb = wc = None
    if warm is not None:
        wa, wb, wc = (_d(w) for w in warm)
    check(lib().orc_wrench_solve(k, _p(p), _p(n), float(lam), float(mu), int(mode),
                                 int(iterations), int(warm_iterations), float(step),
                                 int(max_backtracks), None if wa is None else _p(wa),
                                 None if wb is None else _p(wb), None if wc is None else _p(wc),
                                 C.byref(obj), C.byref(anchor), _p(al), _p(bx), _p(by)))
    return obj.value, anchor.value, al, bx, by


def wrench_objective(points, normals, alpha, bx=None, by=None, lam=10.0, mu=0.0):
    p, n = _d(points).reshape(-1, 3), _d(normals).reshape(-1, 3)
    k = len(p)
    a = _d(alpha)
    bx = np.zeros(k) if bx is None else _d(bx)
    by = np.zeros(k) if by is None else _d(by)
    out = C.c_double()
    check(lib().orc_wrench_objective(k, _p(p), _p(n), float(lam), float(mu), _p(a), _p(bx),
                                     _p(by), C.byref(out)))
    return out.value


def optimize_contacts(domains, statics=(), n_outer=8, n_inner=32, restarts=4, sigma=0.01,
                      lam=10.0, mu=0.3, seed=0):
    """domains: list of (positions (m,3), outward normals (m,3))."""
    counts = np.array([len(d[0]) for d in domains], dtype=np.int32)
    pos = _d(np.concatenate([np.asarray(d[0]).reshape(-1, 3) for d in domains]))
    nrm = _d(np.concatenate([np.asarray(d[1]).reshape(-1, 3) for d in domains]))
    sp = _d(np.array([s[0] for s in statics]).reshape(-1, 3)) if statics else np.zeros((0, 3))
    sn = _d(np.array([s[1] for s in statics]).reshape(-1, 3)) if statics else np.zeros((0, 3))
    ids = np.zeros(len(domains), dtype=np.int32)
    obj = C.c_double()
    ev = C.c_int()
    check(lib().orc_optimize_contacts(len(domains), _i(counts), _p(pos), _p(nrm), len(sp), _p(sp),
                                      _p(sn), n_outer, n_inner, restarts, float(sigma),
                                      float(lam), float(mu), C.c_uint64(seed), _i(ids),
                                      C.byref(obj), C.byref(ev)))
    return ids, obj.value, ev.value


def collision(hand_desc, q, pose12, samples, margin=0.002):
    q, p = _d(q), _d(pose12)
    s = _d(samples).reshape(-1, 6)
    clean, nv = C.c_int(), C.c_int()
    mp = C.c_double()
    check(lib().orc_collision(C.byref(hand_desc), _p(q), _p(p), _p(s), len(s), float(margin),
                              C.byref(clean), C.byref(mp), C.byref(nv)))
    return bool(clean.value), mp.value, nv.value


def gjk(hand_desc, part_a, pose_a, part_b, pose_b):
    pa, pb = _d(pose_a), _d(pose_b)
    d = C.c_double()
    check(lib().orc_gjk(C.byref(hand_desc), int(part_a), _p(pa), int(part_b), _p(pb),
                        C.byref(d)))
    return d.value


def _targets(targets):
    k = len(targets)
    op = _d([t[0] for t in targets]).reshape(k, 3)
    on = _d([t[1] for t in targets]).reshape(k, 3)
    links = np.array([t[2] for t in targets], dtype=np.int32)
    hp = _d([t[3] for t in targets]).reshape(k, 3)
    hn = _d([t[4] for t in targets]).reshape(k, 3)
    return k, op, on, links, hp, hn


def ik(hand_desc, q0, targets, beta=0.01, iterations=30, step_clamp=0.2, residual_tol=1e-4,
       damping_scale=1e-4):
    """targets: list of (object_point, object_normal_inward, link, hand_point, hand_normal)."""
    k, op, on, links, hp, hn = _targets(targets)
    q0 = _d(q0)
    q = np.zeros(hand_desc.dof)
    it, fin = C.c_int(), C.c_int()
    obj = C.c_double()
    used = C.c_ulonglong()
    rp, ra = np.zeros(k), np.zeros(k)
    check(lib().orc_ik(C.byref(hand_desc), _p(q0), k, _p(op), _p(on), _i(links), _p(hp), _p(hn),
                       float(beta), int(iterations), float(step_clamp), float(residual_tol),
                       float(damping_scale), _p(q), C.byref(it), C.byref(obj), C.byref(fin),
                       C.byref(used), _p(rp), _p(ra)))
    return dict(q=q, iterations=it.value, objective=obj.value, finite=bool(fin.value),
                used=used.value, res_pos=rp, res_angle=ra)


def realize(hand_desc, q0, targets, beta=0.01, iterations=30, step_clamp=0.2, residual_tol=1e-4,
            damping_scale=1e-4, rounds=4, fine_iters=10):
    k, op, on, links, hp, hn = _targets(targets)
    q0 = _d(q0)
    q = np.zeros(hand_desc.dof)
    mr = C.c_double()
    fin = C.c_int()
    used = C.c_ulonglong()
    check(lib().orc_realize(C.byref(hand_desc), _p(q0), k, _p(op), _p(on), _i(links), _p(hp),
                            _p(hn), float(beta), int(iterations), float(step_clamp),
                            float(residual_tol), float(damping_scale), int(rounds),
                            int(fine_iters), _p(q), C.byref(mr), C.byref(fin), C.byref(used)))
    return dict(q=q, max_residual=mr.value, finite=bool(fin.value), used=used.value)


class OrcResult:
    def __init__(self, h):
        L = lib()
        self.profile_struct = A.Profile()
        L.orc_result_profile(h, C.byref(self.profile_struct))
        self.profile = {n: getattr(self.profile_struct, n) for n, _ in A.Profile._fields_}
        from paper_2511_07418_b200.api import _copy_structs
        self.grasps = _copy_structs(L.orc_result_grasps(h), L.orc_result_num_grasps(h),
                                    A.grasp_dtype())
        self.traces = _copy_structs(L.orc_result_traces(h), L.orc_result_num_traces(h),
                                    A.trace_dtype())
        L.orc_result_destroy(h)


def run_batch(hand_desc, patches_desc, raw_samples, params, workers=1):
    raw = _d(raw_samples).reshape(-1, 6)
    h = C.c_void_p()
    check(lib().orc_run_batch(C.byref(hand_desc), C.byref(patches_desc), _p(raw), len(raw),
                              C.byref(params), int(workers), C.byref(h)))
    return OrcResult(h)


def run_batch_field(field, hand_desc, patches_desc, raw_samples, params, workers=1):
    """run_batch with a prebuilt OrcField (the reference's cached-index mode)."""
    raw = _d(raw_samples).reshape(-1, 6)
    h = C.c_void_p()
    check(lib().orc_run_batch_field(field._h, C.byref(hand_desc), C.byref(patches_desc), _p(raw),
                                    len(raw), C.byref(params), int(workers), C.byref(h)))
    return OrcResult(h)


def validate(hand_desc, grasps, mesh_verts, mesh_tris, samples, params):
    """validate_dataset restated (validate.cpp:56-175): lg_grasp_check records."""
    g = np.ascontiguousarray(np.asarray(grasps).astype(A.grasp_dtype()))
    v = np.ascontiguousarray(mesh_verts, dtype=np.float64)
    t = np.ascontiguousarray(mesh_tris, dtype=np.int32)
    s = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 6)
    out = np.zeros(len(g), dtype=A.check_dtype())
    check(lib().orc_validate(C.byref(hand_desc), g.ctypes.data_as(C.c_void_p), len(g), _p(v), len(v),
                             t.ctypes.data_as(C.POINTER(C.c_int)), len(t), _p(s), len(s),
                             C.byref(params), out.ctypes.data_as(C.c_void_p)))
    return out
