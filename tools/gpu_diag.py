"""Stage-by-stage device-vs-oracle diagnostics (prints the first mismatches)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import caller as lc
import paper_2511_07418_b200 as lg
from oracle import orc_py as orc

A = os.path.join(ROOT, "assets")
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p = lc.parse_config(f"{A}/configs/four_finger.cfg", hand=f"{A}/hands/four_finger.urdf",
                    object=f"{A}/objects/sphere_r030.obj", batch=batch)
p.passes = 2
p.want_trace = 1
hand, patches, raw, _ = lc.prepare_inputs(p)
ctx = lg.Context(0)
t = time.time()
f = lg.ContactFieldIndex.build(ctx, hand, patches, p.field_configs, p.box_width, p.seed, p.codebook_size)
print("device field build", time.time() - t)
fo = orc.OrcField(hand.desc, patches.desc, p.field_configs, p.box_width, p.seed, p.codebook_size)
ed, eo = f.export(), fo.export()
for k in eo:
    a, b = ed[k], eo[k]
    same = np.array_equal(np.asarray(a), np.asarray(b))
    print(f"field {k}: {'OK' if same else 'MISMATCH'} {np.shape(a)} {np.shape(b)}")
gl, ng = hand.groups()
gop = gl[patches.link_of_patch()]
rng = np.random.default_rng(0)
poses = []
for i in range(8):
    q = rng.normal(size=4); q /= np.linalg.norm(q)
    w, x, y, z = q
    R = np.array([[1-2*(y*y+z*z), 2*(x*y-z*w), 2*(x*z+y*w)], [2*(x*y+z*w), 1-2*(x*x+z*z), 2*(y*z-x*w)], [2*(x*z-y*w), 2*(y*z+x*w), 1-2*(x*x+y*y)]])
    poses.append(np.concatenate([R.ravel(), [0.0, 0.0, 0.05 + 0.01 * i]]))
poses = np.array(poses)
md = lg.query_domains_batch(ctx, f, gop, raw, poses, p.theta_hit)
for i in range(len(poses)):
    mo, so, sz = fo.query(hand.desc, raw, poses[i], p.theta_hit)
    print("query pose", i, "OK" if np.array_equal(md[i], mo) else "MISMATCH", int((mo != 0).sum()))
kd = lg.preprocess_object(ctx, raw, p.probe_half_width, p.probe_depth_threshold)
ko = orc.preprocess(raw, p.probe_half_width, p.probe_depth_threshold)
print("preprocess", "OK" if np.array_equal(kd, ko) else "MISMATCH", kd.sum())
t = time.time()
dev = lg.run_batch(ctx, hand, patches, raw, p)
print("device run_batch wall", time.time() - t)
t = time.time()
dev2 = lg.run_batch(ctx, hand, patches, raw, p)
print("device run_batch warm wall", time.time() - t, dev2.profile)
t = time.time()
ref = orc.run_batch(hand.desc, patches.desc, raw, p, workers=os.cpu_count())
print("oracle run_batch wall", time.time() - t, "cores", os.cpu_count())
print("dev profile", dev.profile)
print("ref profile", ref.profile)
td, tr = dev.traces, ref.traces
print("traces", len(td), len(tr))
bad = 0
for name in tr.dtype.names:
    a, b = td[name], tr[name]
    eq = np.array([np.asarray(x).tobytes() == np.asarray(y).tobytes() for x, y in zip(a, b)])
    if not eq.all():
        idx = np.nonzero(~eq)[0]
        bad += 1
        print(f"trace field {name}: {len(idx)} mismatches, first at {idx[:5]}")
        for j in idx[:2]:
            print("   dev", a[j], "\n   ref", b[j])
print("trace fields mismatching:", bad)
gd, gr = dev.grasps, ref.grasps
print("grasps", len(gd), len(gr), "bitwise equal" if len(gd) == len(gr) and gd.tobytes() == gr.tobytes() else "DIFFER")
