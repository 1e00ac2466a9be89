"""Seed sharding across GPUs and the final gather of valid grasps
(SURVEY.md 8(e)).

Rank r of R owns candidates c in [r*B/R, (r+1)*B/R) for every pass; every
per-candidate RNG stream depends only on (seed, tag, c or g), so the union of
the shards is the single-GPU result.  The only collective is the final
gather of the kept grasps to rank 0, done by the library over NCCL behind the
C-ABI (lg_comm_gather: an all-gather of per-rank headers, then grouped
send/recv of the packed records); rank 0 gets them ordered by
g = pass*batch + c, run_batch's `kept` order (pipeline.cpp:607-614).  The
caller only distributes the 128-byte NCCL id (any transport: torch.distributed
in bench.py, MPI, a shared file).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import lgabi as A


def shard_params(params, rank, world):
    p = A.RunParams()
    C.pointer(p)[0] = params
    p.shard_rank = int(rank)
    p.shard_count = int(world)
    return p


def shard_range(batch, rank, world):
    return batch * rank // world, batch * (rank + 1) // world


class Comm:
    """NCCL communicator of one rank behind the C-ABI (lg_comm_*)."""

    def __init__(self, ctx, rank, world, uid):
        from .api import lib, check
        L = lib()
        self._ctx = ctx
        self.rank, self.world = int(rank), int(world)
        buf = (C.c_ubyte * A.LG_COMM_ID_BYTES).from_buffer_copy(bytes(uid))
        self._h = C.c_void_p()
        check(L.lg_comm_init(ctx._h, buf, self.rank, self.world, C.byref(self._h)))

    @staticmethod
    def unique_id():
        from .api import lib, check
        buf = (C.c_ubyte * A.LG_COMM_ID_BYTES)()
        check(lib().lg_comm_unique_id(buf))
        return bytes(buf)

    def gather(self, result):
        """Rank 0: (all grasps in g order, merged profile dict); else (None, None)."""
        from .api import lib, check, _copy_structs
        g = np.ascontiguousarray(result.grasps)
        out = C.POINTER(A.Grasp)()
        n_all = C.c_longlong(0)
        merged = A.Profile()
        check(lib().lg_comm_gather(self._h, g.ctypes.data_as(C.POINTER(A.Grasp)), len(g),
                                   C.byref(result.profile_struct), C.byref(out), C.byref(n_all),
                                   C.byref(merged)))
        if self.rank != 0:
            return None, None
        grasps = _copy_structs(out, n_all.value, A.grasp_dtype())
        return grasps, {n: getattr(merged, n) for n, _ in A.Profile._fields_}

    def close(self):
        from .api import lib
        if self._h:
            lib().lg_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def merge_grasps(grasps):
    """Order gathered grasps by candidate id g (pipeline.cpp:607-614)."""
    if len(grasps) == 0:
        return grasps
    return grasps[np.argsort(grasps["g"], kind="stable")]


def sum_profiles(profiles):
    """Funnel counts add across shards; stage times are the max over ranks."""
    out = dict(profiles[0])
    for p in profiles[1:]:
        for k, v in p.items():
            if k in ("placement_domains", "contact_optimization", "kinematics_optimization",
                     "postprocessing", "total", "field_build"):
                out[k] = max(out[k], v)
            elif k in ("patches", "boxes", "field_vectors", "object_samples", "field_samples"):
                out[k] = v
            else:
                out[k] = out[k] + v
    out["grasps_per_second"] = out["valid"] / out["total"] if out["total"] > 0 else 0.0
    return out
