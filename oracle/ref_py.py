"""ctypes binding of the REFERENCE ITSELF (oracle/_ref/libgraspgen_ref.so:
/root/reference/proj/src compiled unmodified against oracle/shim, plus the C
entry points of oracle/ref_capi.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product path.
The library is prebuilt by `make -C oracle` (run from __graft_entry__.build()
where /root/reference exists) and travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2511_07418_b200 import lgabi as A

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
LIB_PATH = os.path.join(REF_DIR, "libgraspgen_ref.so")
_LIB = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle ref` where "
                               "/root/reference exists")
        L = C.CDLL(LIB_PATH)
        vp, P, dp, ip, llp = C.c_void_p, C.POINTER, A.dp, A.ip, A.llp
        u64 = C.c_uint64
        sig = {
            "ref_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
            "ref_prepare": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                      C.c_longlong, C.c_int, C.c_int, P(vp)]),
            "ref_inputs_destroy": (None, [vp]),
            "ref_params": (C.c_int, [vp, P(A.RunParams)]),
            "ref_hand_desc": (C.c_int, [vp, P(A.HandDesc)]),
            "ref_patches_desc": (C.c_int, [vp, P(A.PatchesDesc)]),
            "ref_raw_samples": (C.c_int, [vp, P(dp), ip]),
            "ref_groups": (C.c_int, [vp, ip, ip, ip]),
            "ref_link_name": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t]),
            "ref_link_visual": (C.c_int, [vp, C.c_int, ip, ip, dp, ip]),
            "ref_index_cache_key": (C.c_int, [vp, P(u64)]),
            "ref_run_batch": (C.c_int, [vp, P(vp)]),
            "ref_hand_load": (C.c_int, [C.c_char_p, C.c_double, P(vp)]),
            "ref_hand_desc_of": (C.c_int, [vp, P(A.HandDesc)]),
            "ref_hand_visual": (C.c_int, [vp, P(ip), P(dp), P(ip), P(ip), P(ip), ip]),
            "ref_hand_link_name": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t]),
            "ref_hand_joint_name": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t]),
            "ref_hand_destroy": (None, [vp]),
            "ref_result_num_grasps": (C.c_longlong, [vp]),
            "ref_result_grasps": (vp, [vp]),
            "ref_result_profile": (C.c_int, [vp, P(A.Profile)]),
            "ref_result_extras": (C.c_int, [vp] + [llp] * 7),
            "ref_result_destroy": (None, [vp]),
            "ref_field_build": (C.c_int, [vp, C.c_int, P(vp)]),
            "ref_field_export": (C.c_int, [vp, P(A.FieldCsr)]),
            "ref_field_save": (C.c_int, [vp, C.c_char_p, u64]),
            "ref_field_memory_bytes": (C.c_longlong, [vp]),
            "ref_field_destroy": (None, [vp]),
            "ref_preprocess": (C.c_int, [dp, C.c_int, C.c_double, C.c_double, P(C.c_uint8)]),
            "ref_query_domains": (C.c_int, [vp, vp, dp, C.c_int, dp, C.c_double, ip, ip, llp, llp,
                                            C.c_longlong, C.c_longlong, dp, dp, dp, llp, ip, ip]),
            "ref_reverse_lookup": (C.c_int, [vp, C.c_int, ip, ip, dp, dp, u64, ip, dp, dp]),
            "ref_place": (C.c_int, [vp, dp, C.c_int, u64, dp, ip, dp, ip, dp, dp, ip]),
            "ref_optimize_contacts": (C.c_int, [C.c_int, ip, dp, dp, C.c_int, dp, dp, C.c_int,
                                                C.c_int, C.c_int, C.c_double, C.c_double,
                                                C.c_double, C.c_int, C.c_int, C.c_double, u64, ip,
                                                dp, ip, dp, dp, dp, ip, ip]),
            "ref_wrench_solve": (C.c_int, [C.c_int, dp, dp, C.c_double, C.c_double, C.c_int,
                                           C.c_int, C.c_int, C.c_double, dp, ip, dp, dp, dp]),
            "ref_realize": (C.c_int, [vp, dp, C.c_int, dp, dp, ip, dp, dp, C.c_double, C.c_int,
                                      C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, dp, dp,
                                      ip, P(C.c_ulonglong), dp, dp, ip, dp]),
            "ref_collision": (C.c_int, [vp, dp, dp, dp, C.c_int, C.c_double, ip, dp, ip, C.c_int,
                                        ip, ip, dp, ip]),
            "ref_contact_ik": (C.c_int, [vp, dp, C.c_int, dp, dp, ip, dp, dp, C.c_double, C.c_int,
                                         C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                         dp, ip, P(C.c_ulonglong), ip, dp, dp, dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


class RefError(RuntimeError):
    pass


def check(rc):
    if rc != 0:
        buf = C.create_string_buffer(4096)
        lib().ref_last_error(buf, len(buf))
        raise RefError(f"reference error {rc}: {buf.value.decode()}")


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(A.dp)


def _i(a):
    return a.ctypes.data_as(A.ip)


class RefInputs:
    """The reference's own inputs for one run: parse_config + build_field's and
    run_batch's host steps (pipeline.cpp:273-331), exported in the lg.h
    descriptor layout (hand_desc, patches_desc, raw samples, params)."""

    def __init__(self, config=None, extra="", hand=None, object=None, out=None, seed=None,
                 batch=None, workers=None):
        L = lib()
        self._h = C.c_void_p()
        enc = (lambda s: None if s is None else str(s).encode())
        check(L.ref_prepare(enc(config), enc(extra), enc(hand), enc(object), enc(out),
                            -1 if seed is None else int(seed), -1 if batch is None else int(batch),
                            -1 if workers is None else int(workers), C.byref(self._h)))
        self.params = A.RunParams()
        check(L.ref_params(self._h, C.byref(self.params)))
        self.hand_desc = A.HandDesc()
        check(L.ref_hand_desc(self._h, C.byref(self.hand_desc)))
        self.patches_desc = A.PatchesDesc()
        check(L.ref_patches_desc(self._h, C.byref(self.patches_desc)))
        ptr, n = A.dp(), C.c_int(0)
        check(L.ref_raw_samples(self._h, C.byref(ptr), C.byref(n)))
        self.raw = np.ctypeslib.as_array(ptr, shape=(n.value, 6)).copy() if n.value else \
            np.zeros((0, 6))
        nl = self.hand_desc.n_links
        self.group_of_link = np.zeros(nl, dtype=np.int32)
        self.group_of_patch = np.zeros(max(1, self.patches_desc.n_patches), dtype=np.int32)
        ng = C.c_int(0)
        check(L.ref_groups(self._h, _i(self.group_of_link), _i(self.group_of_patch), C.byref(ng)))
        self.group_of_patch = self.group_of_patch[:self.patches_desc.n_patches]
        self.n_groups = ng.value

    def close(self):
        if self._h:
            lib().ref_inputs_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def link_name(self, link):
        buf = C.create_string_buffer(256)
        check(lib().ref_link_name(self._h, int(link), buf, len(buf)))
        return buf.value.decode()

    def link_visual(self, link):
        nv, nt = C.c_int(0), C.c_int(0)
        check(lib().ref_link_visual(self._h, int(link), C.byref(nv), C.byref(nt), None, None))
        v = np.zeros((nv.value, 3))
        t = np.zeros((nt.value, 3), dtype=np.int32)
        check(lib().ref_link_visual(self._h, int(link), C.byref(nv), C.byref(nt), _p(v), _i(t)))
        return v, t

    def cache_key(self):
        k = C.c_uint64(0)
        check(lib().ref_index_cache_key(self._h, C.byref(k)))
        return k.value

    def run_batch(self):
        """The reference's run_batch(cfg) — its own loaders, field build and
        four-stage pass, with cfg.workers threads."""
        return RefResult(self)

    def field(self, N=0):
        return RefField(self, N)


def load_hand_arrays(urdf, scale=1.0):
    """The reference's load_hand + dependency_groups as plain numpy arrays
    (lg_hand_desc fields, visual meshes, link names, group ids)."""
    L = lib()
    h = C.c_void_p()
    check(L.ref_hand_load(str(urdf).encode(), float(scale), C.byref(h)))
    try:
        d = A.HandDesc()
        check(L.ref_hand_desc_of(h, C.byref(d)))
        nl, npart = d.n_links, d.n_parts

        def arr(ptr, n, dt):
            return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt).copy() if n else np.zeros(0, dt)

        out = {"n_links": nl, "dof": d.dof, "root": d.root,
               "parent": arr(d.parent, nl, np.int32), "joint_type": arr(d.joint_type, nl, np.int32),
               "joint_index": arr(d.joint_index, nl, np.int32),
               "topo_order": arr(d.topo_order, nl, np.int32),
               "origin_R": arr(d.origin_R, 9 * nl, np.float64),
               "origin_t": arr(d.origin_t, 3 * nl, np.float64),
               "axis": arr(d.axis, 3 * nl, np.float64),
               "limit_lo": arr(d.limit_lo, nl, np.float64), "limit_hi": arr(d.limit_hi, nl, np.float64),
               "part_link": arr(d.part_link, npart, np.int32),
               "part_vert_off": arr(d.part_vert_off, npart + 1, np.int32),
               "part_tri_off": arr(d.part_tri_off, npart + 1, np.int32),
               "part_plane_off": arr(d.part_plane_off, npart + 1, np.int32)}
        out["part_verts"] = arr(d.part_verts, 3 * int(out["part_vert_off"][-1]), np.float64)
        out["part_tris"] = arr(d.part_tris, 3 * int(out["part_tri_off"][-1]), np.int32)
        out["part_planes"] = arr(d.part_planes, 4 * int(out["part_plane_off"][-1]), np.float64)
        out["part_bounds"] = arr(d.part_bounds, 6 * npart, np.float64)
        vo, vv, to, tt, gl = A.ip(), A.dp(), A.ip(), A.ip(), A.ip()
        ng = C.c_int(0)
        check(L.ref_hand_visual(h, C.byref(vo), C.byref(vv), C.byref(to), C.byref(tt), C.byref(gl),
                                C.byref(ng)))
        out["vis_vert_off"] = arr(vo, nl + 1, np.int32)
        out["vis_tri_off"] = arr(to, nl + 1, np.int32)
        out["vis_verts"] = arr(vv, 3 * int(out["vis_vert_off"][-1]), np.float64)
        out["vis_tris"] = arr(tt, 3 * int(out["vis_tri_off"][-1]), np.int32)
        out["group_of_link"] = arr(gl, nl, np.int32)
        out["n_groups"] = ng.value
        names, jnames = [], []
        for l in range(nl):
            buf = C.create_string_buffer(256)
            check(L.ref_hand_link_name(h, l, buf, len(buf)))
            names.append(buf.value.decode())
            check(L.ref_hand_joint_name(h, l, buf, len(buf)))
            jnames.append(buf.value.decode())
        out["link_names"] = np.array(names)
        out["joint_names"] = np.array(jnames)
        return out
    finally:
        L.ref_hand_destroy(h)


class RefResult:
    def __init__(self, inputs):
        L = lib()
        h = C.c_void_p()
        check(L.ref_run_batch(inputs._h, C.byref(h)))
        self.profile_struct = A.Profile()
        check(L.ref_result_profile(h, C.byref(self.profile_struct)))
        self.profile = {n: getattr(self.profile_struct, n) for n, _ in A.Profile._fields_}
        n = L.ref_result_num_grasps(h)
        dt = A.grasp_dtype()
        if n:
            buf = (C.c_char * (n * dt.itemsize)).from_address(L.ref_result_grasps(h))
            self.grasps = np.frombuffer(bytes(buf), dtype=dt).copy()
        else:
            self.grasps = np.zeros(0, dtype=dt)
        ex = [C.c_longlong(0) for _ in range(7)]
        check(L.ref_result_extras(h, *[C.byref(e) for e in ex]))
        (self.index_memory_bytes, self.hand_links, self.hand_joints, self.hand_parts,
         self.triangles_read, self.triangles_kept, self.degenerate_dropped) = [e.value for e in ex]
        L.ref_result_destroy(h)


class RefField:
    """ContactFieldIndex::build (contact_field.cpp:306-334) on the reference
    inputs, with lg.h CSR export."""

    def __init__(self, inputs, N=0):
        self.inputs = inputs
        self._h = C.c_void_p()
        check(lib().ref_field_build(inputs._h, int(N), C.byref(self._h)))
        self.csr = A.FieldCsr()
        check(lib().ref_field_export(self._h, C.byref(self.csr)))

    def close(self):
        if self._h:
            lib().ref_field_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def save(self, path, key):
        check(lib().ref_field_save(self._h, str(path).encode(), int(key)))

    def memory_bytes(self):
        return lib().ref_field_memory_bytes(self._h)

    def query(self, samples, pose12, theta_hit):
        """query_domains for one pose -> list over groups of element dicts
        {pos, nrm, score, hits: [(patch, box), ...]} in sample order."""
        s = _d(samples).reshape(-1, 6)
        pose = _d(pose12).reshape(12)
        L = lib()
        ng = C.c_int(0)
        n_elem = np.zeros(64, dtype=np.int32)
        te, th = C.c_longlong(0), C.c_longlong(0)
        args = (self._h, self.inputs._h, _p(s), len(s), _p(pose), float(theta_hit), C.byref(ng),
                _i(n_elem), C.byref(te), C.byref(th))
        check(L.ref_query_domains(*args, 0, 0, None, None, None, None, None, None))
        E, H = te.value, th.value
        pos, nrm, score = np.zeros((E, 3)), np.zeros((E, 3)), np.zeros(E)
        off = np.zeros(E + 1, dtype=np.int64)
        hp, hb = np.zeros(max(H, 1), dtype=np.int32), np.zeros(max(H, 1), dtype=np.int32)
        check(L.ref_query_domains(*args, E, H, _p(pos), _p(nrm), _p(score),
                                  off.ctypes.data_as(A.llp), _i(hp), _i(hb)))
        out, k = [], 0
        for g in range(ng.value):
            els = []
            for _ in range(n_elem[g]):
                hits = list(zip(hp[off[k]:off[k + 1]].tolist(), hb[off[k]:off[k + 1]].tolist()))
                els.append({"pos": pos[k], "nrm": nrm[k], "score": score[k], "hits": hits})
                k += 1
            out.append(els)
        return out

    def reverse_lookup(self, element, seed):
        hits = element["hits"]
        hp = np.array([h[0] for h in hits], dtype=np.int32)
        hb = np.array([h[1] for h in hits], dtype=np.int32)
        link = C.c_int(0)
        pt, nr = np.zeros(3), np.zeros(3)
        check(lib().ref_reverse_lookup(self._h, len(hits), _i(hp), _i(hb), _p(_d(element["pos"])),
                                       _p(_d(element["nrm"])), int(seed), C.byref(link), _p(pt),
                                       _p(nr)))
        return link.value, pt, nr


def preprocess(samples, h, d):
    s = _d(samples).reshape(-1, 6)
    keep = np.zeros(len(s), dtype=np.uint8)
    check(lib().ref_preprocess(_p(s), len(s), float(h), float(d),
                               keep.ctypes.data_as(C.POINTER(C.c_uint8))))
    return keep


def place(inputs, field_samples, seed):
    s = _d(field_samples).reshape(-1, 6)
    pose = np.zeros(12)
    acc, pen, ns = C.c_int(0), C.c_double(0), C.c_int(0)
    sp, sn = np.zeros((4, 3)), np.zeros((4, 3))
    sl = np.zeros(4, dtype=np.int32)
    check(lib().ref_place(inputs._h, _p(s), len(s), int(seed), _p(pose), C.byref(acc),
                          C.byref(pen), C.byref(ns), _p(sp), _p(sn), _i(sl)))
    n = ns.value
    return {"pose": pose, "accepted": acc.value, "penetration": pen.value,
            "static_p": sp[:n].copy(), "static_n": sn[:n].copy(), "static_link": sl[:n].copy()}


def optimize_contacts(domains, statics=(), n_outer=8, n_inner=32, restarts=4, sigma=0.01,
                      lambda_torque=10.0, mu=0.3, iterations=64, warm_iterations=8, step=0.1,
                      seed=0):
    """optimize_contacts over k domains given as (positions [n,3], normals [n,3])."""
    k = len(domains)
    dn = np.array([len(p) for p, _ in domains], dtype=np.int32)
    dp_ = _d(np.concatenate([np.asarray(p).reshape(-1, 3) for p, _ in domains]))
    dnr = _d(np.concatenate([np.asarray(n).reshape(-1, 3) for _, n in domains]))
    ns = len(statics)
    sp = _d([s[0] for s in statics]).reshape(-1, 3) if ns else np.zeros((1, 3))
    sn = _d([s[1] for s in statics]).reshape(-1, 3) if ns else np.zeros((1, 3))
    ids = np.zeros(k, dtype=np.int32)
    obj, anc, ev, val = C.c_double(0), C.c_int(0), C.c_int(0), C.c_int(0)
    al, bx, by = np.zeros(k + ns), np.zeros(k + ns), np.zeros(k + ns)
    check(lib().ref_optimize_contacts(k, _i(dn), _p(dp_), _p(dnr), ns, _p(sp), _p(sn), n_outer,
                                      n_inner, restarts, sigma, lambda_torque, mu, iterations,
                                      warm_iterations, step, int(seed), _i(ids), C.byref(obj),
                                      C.byref(anc), _p(al), _p(bx), _p(by), C.byref(ev),
                                      C.byref(val)))
    return {"element_ids": ids, "objective": obj.value, "anchor": anc.value, "alpha": al,
            "beta_x": bx, "beta_y": by, "evaluations": ev.value, "valid": val.value}


def wrench_solve(points, normals, lambda_torque=10.0, mu=0.0, gswo=False, iterations=64,
                 warm_iterations=8, step=0.1):
    p, n = _d(points).reshape(-1, 3), _d(normals).reshape(-1, 3)
    m = len(p)
    obj, anc = C.c_double(0), C.c_int(0)
    al, bx, by = np.zeros(m), np.zeros(m), np.zeros(m)
    check(lib().ref_wrench_solve(m, _p(p), _p(n), lambda_torque, mu, int(bool(gswo)), iterations,
                                 warm_iterations, step, C.byref(obj), C.byref(anc), _p(al), _p(bx),
                                 _p(by)))
    return {"objective": obj.value, "anchor": anc.value, "alpha": al, "beta_x": bx, "beta_y": by}


def realize(inputs, q0, targets, beta=0.01, iterations=30, step_clamp=0.2, residual_tol=1e-4,
            damping_scale=1e-4, finetune_rounds=4, finetune_iterations=10):
    """realize_grasp; targets = [(obj_p, obj_n, link, hand_p, hand_n), ...]."""
    k = len(targets)
    op = _d([t[0] for t in targets]).reshape(-1, 3)
    on = _d([t[1] for t in targets]).reshape(-1, 3)
    lk = np.array([t[2] for t in targets], dtype=np.int32)
    hp = _d([t[3] for t in targets]).reshape(-1, 3)
    hn = _d([t[4] for t in targets]).reshape(-1, 3)
    dof = inputs.hand_desc.dof
    q = np.zeros(dof)
    mr, fin, used = C.c_double(0), C.c_int(0), C.c_ulonglong(0)
    rp, rn = np.zeros((k, 3)), np.zeros((k, 3))
    rl, res = np.zeros(k, dtype=np.int32), np.zeros(k)
    check(lib().ref_realize(inputs._h, _p(_d(q0)), k, _p(op), _p(on), _i(lk), _p(hp), _p(hn), beta,
                            iterations, step_clamp, residual_tol, damping_scale, finetune_rounds,
                            finetune_iterations, _p(q), C.byref(mr), C.byref(fin), C.byref(used),
                            _p(rp), _p(rn), _i(rl), _p(res)))
    return {"q": q, "max_residual": mr.value, "finite": fin.value, "used_joints": used.value,
            "realized_p": rp, "realized_n": rn, "realized_link": rl, "residuals": res}


def contact_ik(inputs, q0, targets, beta=0.01, iterations=30, step_clamp=0.2, residual_tol=1e-4,
               damping_scale=1e-4, damping_min=1e-6, max_backtracks=10):
    """solve_contact_ik; targets = [(obj_p, obj_n, link, hand_p, hand_n), ...]."""
    k = len(targets)
    op = _d([t[0] for t in targets]).reshape(-1, 3)
    on = _d([t[1] for t in targets]).reshape(-1, 3)
    lk = np.array([t[2] for t in targets], dtype=np.int32)
    hp = _d([t[3] for t in targets]).reshape(-1, 3)
    hn = _d([t[4] for t in targets]).reshape(-1, 3)
    q = np.zeros(inputs.hand_desc.dof)
    fin, used, its, obj = C.c_int(0), C.c_ulonglong(0), C.c_int(0), C.c_double(0)
    pos, ang = np.zeros(max(k, 1)), np.zeros(max(k, 1))
    check(lib().ref_contact_ik(inputs._h, _p(_d(q0)), k, _p(op), _p(on), _i(lk), _p(hp), _p(hn),
                               beta, iterations, step_clamp, residual_tol, damping_scale,
                               damping_min, max_backtracks, _p(q), C.byref(fin), C.byref(used),
                               C.byref(its), C.byref(obj), _p(pos), _p(ang)))
    return {"q": q, "finite": fin.value, "used_joints": used.value, "iterations": its.value,
            "objective": obj.value, "position": pos[:k], "normal_angle": ang[:k]}


def collision(inputs, q, pose12, samples, margin=0.002, cap=256):
    s = _d(samples).reshape(-1, 6)
    clean, mp, nv, bp = C.c_int(0), C.c_double(0), C.c_int(0), C.c_int(0)
    va, vb = np.zeros(cap, dtype=np.int32), np.zeros(cap, dtype=np.int32)
    vd = np.zeros(cap)
    check(lib().ref_collision(inputs._h, _p(_d(q)), _p(_d(pose12)), _p(s), len(s), float(margin),
                              C.byref(clean), C.byref(mp), C.byref(nv), cap, _i(va), _i(vb),
                              _p(vd), C.byref(bp)))
    n = min(nv.value, cap)
    return {"clean": clean.value, "max_penetration": mp.value, "n_violations": nv.value,
            "broad_pairs": bp.value,
            "violations": list(zip(va[:n].tolist(), vb[:n].tolist(), vd[:n].tolist()))}
