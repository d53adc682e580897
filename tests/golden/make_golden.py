"""Generate golden fixtures by running the REFERENCE (octrf) in this container.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The reference is only importable in the build
container; the fixtures travel, the reference does not.  Every fixture holds
the reference's *inputs* in its own pool layout (child/parent/depth/leaf/
alive/center/sigma/sh/free list) so tests can rebuild the exact tree without
octrf, plus the reference's outputs from its public API:
segment_batch, render_rays(return_aux=True), render_and_backprop, calibrate
(+ the .dot1 sha256 of the canonicalised result), and the config-1 scene.
"""

from __future__ import annotations

import hashlib
import io
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import octrf  # noqa: E402
from octrf import LeafPayload, build_dense, save_tree, load_tree  # noqa: E402
from octrf.calibrate import CalibrationConfig, calibrate, select_prune, select_sample  # noqa: E402
from octrf.render import render_and_backprop, render_rays, segment_batch  # noqa: E402
from octrf.signals import SignalBuffer, SignalTarget  # noqa: E402
from octrf.scene_io import Camera  # noqa: E402

from paper_2307_15333_b200 import scenes  # noqa: E402


def pool_arrays(tree, prefix=""):
    return {
        prefix + "child": tree._child.copy(), prefix + "parent": tree._parent.copy(),
        prefix + "depth": tree._depth.copy(), prefix + "leaf": tree._leaf.copy(),
        prefix + "alive": tree._alive.copy(), prefix + "center": tree._center.copy(),
        prefix + "sigma": tree.sigma.copy(), prefix + "sh": tree.sh.copy(),
        prefix + "free": np.asarray(tree._free, dtype=np.int64),
        prefix + "root_center": tree.center.copy(),
        prefix + "half_extent": np.float64(tree.half_extent),
        prefix + "basis_count": np.int64(tree.basis_count),
        prefix + "max_depth": np.int64(tree.max_depth),
    }


def dot1_bytes(tree) -> bytes:
    path = "/tmp/_golden_tmp.dot1"
    save_tree(tree, path)
    with open(path, "rb") as fh:
        return fh.read()


def irregular_tree(seed, depth=2, basis_count=1, splits=6, merges=3, resplits=2,
                   center=(0.0, 0.0, 0.0), half=1.0, max_depth=4, sigma_range=(0.05, 5.0)):
    """Seeded irregular pool tree: dense build, random splits, merges (which
    free slots), then more splits that reuse those slots LIFO."""
    rng = np.random.default_rng(seed)
    nsh = 3 * basis_count

    def init(c):
        return rng.uniform(*sigma_range, len(c)), rng.normal(0.0, 1.0, (len(c), nsh))

    tree = build_dense(depth, center, half, basis_count, init, max_depth=max_depth)

    def split_some(k):
        for _ in range(k):
            leaves = tree.leaf_ids()
            ok = leaves[tree._depth[leaves] < max_depth]
            if ok.size == 0:
                return
            kids = tree.split_leaf(int(rng.choice(ok)))
            tree.sigma[kids] = rng.uniform(*sigma_range, 8).astype(np.float32)
            tree.sh[kids] = rng.normal(0.0, 1.0, (8, nsh)).astype(np.float32)

    split_some(splits)
    for _ in range(merges):
        ints = tree.internal_ids()
        ok = [int(n) for n in ints if tree._leaf[tree._child[n]].all()]
        if not ok:
            break
        tree.merge_children(int(rng.choice(ok)))
    split_some(resplits)
    return tree


def ray_set(seed, n, center=(0.0, 0.0, 0.0), half=1.0, miss_fraction=0.1, specials=True):
    """Seeded rays through the cube, some misses, plus degenerate specials:
    axis-aligned directions (zero components), origins inside the cube,
    origins exactly on a centre plane, rays grazing a face."""
    rng = np.random.default_rng(seed)
    c = np.asarray(center, dtype=np.float64)
    u = rng.normal(0.0, 1.0, (n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    origins = c + u * (3.0 * half)
    target = c + rng.uniform(-0.9, 0.9, (n, 3)) * half
    dirs = target - origins
    k = int(n * miss_fraction)
    if k:
        dirs[:k] = rng.normal(0.0, 1.0, (k, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    if specials:
        sp_o, sp_d = [], []
        for ax in range(3):
            for sgn in (1.0, -1.0):
                o = c + rng.uniform(-0.7, 0.7, 3) * half
                o[ax] = c[ax] - sgn * 2.0 * half
                d = np.zeros(3); d[ax] = sgn
                sp_o.append(o); sp_d.append(d)
        # origin on the root centre planes, axis aligned
        sp_o.append(c + np.array([-2.0 * half, 0.0, 0.0])); sp_d.append(np.array([1.0, 0.0, 0.0]))
        sp_o.append(c + np.array([0.0, 0.0, -2.0 * half])); sp_d.append(np.array([0.0, 0.0, 1.0]))
        # origins inside the cube
        for _ in range(4):
            o = c + rng.uniform(-0.5, 0.5, 3) * half
            d = rng.normal(0.0, 1.0, 3); d /= np.linalg.norm(d)
            sp_o.append(o); sp_d.append(d)
        # diagonal through the centre and a grazing ray on the max face (misses: half-open)
        d = np.ones(3) / np.sqrt(3.0)
        sp_o.append(c - 2.0 * half * d); sp_d.append(d)
        sp_o.append(c + np.array([-2.0 * half, half, 0.0])); sp_d.append(np.array([1.0, 0.0, 0.0]))
        sp_o.append(c + np.array([-2.0 * half, -half, 0.1 * half])); sp_d.append(np.array([1.0, 0.0, 0.0]))
        origins = np.concatenate([origins, np.array(sp_o)])
        dirs = np.concatenate([dirs, np.array(sp_d)])
    return origins, dirs


def render_case(name, tree, origins, dirs, seed, bg, t_near=0.0, t_far=np.inf):
    rng = np.random.default_rng(seed)
    targets = rng.uniform(0.0, 1.0, (origins.shape[0], 3))
    out = dict(pool_arrays(tree))
    out.update(origins=origins, dirs=dirs, targets=targets, bg=np.asarray(bg, dtype=np.float64) * np.ones(3),
               t_near=np.float64(t_near), t_far=np.float64(t_far))
    off, leaf, t, delta = segment_batch(tree, origins, dirs, t_near, t_far)
    out.update(seg_offsets=off, seg_leaf=leaf, seg_t=t, seg_delta=delta)
    for tag, eps in (("eps", 1e-4), ("noeps", 0.0)):
        rgb, tfin, wsum = render_rays(tree, origins, dirs, bg, early_stop_eps=eps,
                                      t_near=t_near, t_far=t_far, return_aux=True)
        out.update({f"rgb_{tag}": rgb, f"tfin_{tag}": tfin, f"wsum_{tag}": wsum})
        loss, grads, signal = render_and_backprop(tree, origins, dirs, targets, bg,
                                                  early_stop_eps=eps, t_near=t_near, t_far=t_far)
        out.update({f"loss_{tag}": np.float64(loss), f"dsigma_{tag}": grads.dsigma,
                    f"dsh_{tag}": grads.dsh, f"touched_{tag}": grads.touched,
                    f"signal_{tag}": signal})
    np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **out)
    print("render", name, "rays", origins.shape[0], "segments", int(off[-1]),
          "cap", tree.capacity)


def calib_case(name, tree, acc, tau, gamma, recursive, threshold=None, target="q"):
    out = dict(pool_arrays(tree))
    tgt = SignalTarget.RAY_WEIGHT_Q if target == "q" else SignalTarget.DENSITY_SIGMA
    buf = SignalBuffer(tree, tgt)
    buf.accumulator[:] = acc
    buf.epoch_rays = 1
    out.update(acc=acc.copy(), tau=np.float64(tau), gamma=np.float64(gamma),
               recursive=np.int64(recursive),
               threshold=np.float64(np.nan if threshold is None else threshold),
               target=np.array(target))
    out["sel_prune"] = select_prune(tree, buf, tau)
    out["sel_sample_pre"] = select_sample(tree, buf, gamma, threshold)
    report = calibrate(tree, buf, CalibrationConfig(tau=tau, gamma=gamma, recursive=recursive,
                                                    sample_threshold=threshold,
                                                    check_invariants=True))
    merges = [(n, k) for kind, n, k in report.events if kind == "merge"]
    splits = [(n, k) for kind, n, k in report.events if kind == "split"]
    out.update(leaves_before=np.int64(report.leaves_before),
               leaves_after=np.int64(report.leaves_after),
               merges_applied=np.int64(report.merges_applied),
               splits_applied=np.int64(report.splits_applied),
               recursion_rounds=np.int64(report.recursion_rounds),
               merge_parents=np.array([m[0] for m in merges], dtype=np.int64),
               split_leaves=np.array([s[0] for s in splits], dtype=np.int64),
               split_kids=np.array([s[1] for s in splits], dtype=np.int64).reshape(-1, 8))
    out.update(pool_arrays(tree, prefix="after_"))
    blob = dot1_bytes(tree)
    out["after_dot1_sha256"] = np.array(hashlib.sha256(blob).hexdigest())
    np.savez_compressed(os.path.join(HERE, f"calib_{name}.npz"), **out)
    print("calib", name, report.to_json())


def config1():
    """BASELINE.json configs[0] through the reference's own API."""
    field = scenes.config1_field()

    def init(c):
        return field.sigma_exact(c), np.zeros((len(c), 12))

    tree = build_dense(5, (0.0, 0.0, 0.0), 1.0, 4, init, max_depth=5)
    buf = SignalBuffer(tree, SignalTarget.DENSITY_SIGMA)
    from octrf.calibrate import prune
    prune(tree, buf, 0.1, recursive=True)
    save_tree(tree, "/tmp/_c1.dot1")
    tree = load_tree("/tmp/_c1.dot1")
    leaves = tree.leaf_ids()
    rng = np.random.default_rng(2)
    tree.sh[leaves] = rng.normal(0.0, 0.3, (leaves.size, 12)).astype(np.float32)
    scene_blob = dot1_bytes(tree)
    focal = scenes.focal_from_angle(64, scenes.FOV_40)
    cam = Camera(64, 64, focal, scenes.orbit_pose(**scenes.CONFIG1_POSE))
    origins, dirs = cam.rays()
    pert = load_tree("/tmp/_c1.dot1")
    pert.sigma[:] = tree.sigma
    pert.sh[leaves] = tree.sh[leaves] + rng.normal(0.0, 0.05, (leaves.size, 12)).astype(np.float32)
    targets = render_rays(pert, origins, dirs, 1.0)
    off, leaf, t, delta = segment_batch(tree, origins, dirs)
    rgb, tfin, wsum = render_rays(tree, origins, dirs, 1.0, return_aux=True)
    loss, grads, signal = render_and_backprop(tree, origins, dirs, targets, 1.0)
    out = dict(scene_sha256=np.array(hashlib.sha256(scene_blob).hexdigest()),
               scene_dot1=np.frombuffer(scene_blob, dtype=np.uint8),
               origins=origins, dirs=dirs, targets=targets, seg_offsets=off,
               seg_leaf=leaf.astype(np.int32), seg_t=t, seg_delta=delta, rgb=rgb, tfin=tfin,
               wsum=wsum, loss=np.float64(loss), touched=grads.touched,
               dsigma_touched=grads.dsigma[grads.touched], dsh_touched=grads.dsh[grads.touched],
               signal=signal)
    buf = SignalBuffer(tree)
    buf.accumulate(signal, origins.shape[0])
    report = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=0.05, recursive=False))
    blob = dot1_bytes(tree)
    out.update(calib_sha256=np.array(hashlib.sha256(blob).hexdigest()),
               calib_merges=np.int64(report.merges_applied),
               calib_splits=np.int64(report.splits_applied),
               calib_leaves_after=np.int64(report.leaves_after))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)
    print("config1 leaves", leaves.size, "segments", int(off[-1]), report.to_json())


def main():
    # --- render / backward cases -------------------------------------------------
    t = irregular_tree(11, depth=2, basis_count=1, splits=8, merges=3, resplits=3, max_depth=4)
    o, d = ray_set(12, 160)
    render_case("b1_irregular", t, o, d, 13, 1.0)
    render_case("b1_window", t, o, d, 14, (0.2, 0.5, 0.8), t_near=2.3, t_far=3.4)
    t = irregular_tree(21, depth=2, basis_count=4, splits=10, merges=2, resplits=2,
                       center=(0.3, -0.2, 0.05), half=1.7, max_depth=4)
    o, d = ray_set(22, 160, center=(0.3, -0.2, 0.05), half=1.7)
    render_case("b4_offcenter", t, o, d, 23, 0.0)
    t = irregular_tree(31, depth=3, basis_count=9, splits=12, merges=4, resplits=4,
                       max_depth=5, sigma_range=(0.0, 3.0))
    o, d = ray_set(32, 200)
    render_case("b9_depth3", t, o, d, 33, (0.9, 0.5, 0.1))
    t = irregular_tree(41, depth=2, basis_count=16, splits=6, merges=1, resplits=2,
                       max_depth=4, sigma_range=(0.0, 40.0))
    o, d = ray_set(42, 160)
    render_case("b16_opaque", t, o, d, 43, 1.0)
    t = build_dense(0, (0.0, 0.0, 0.0), 1.0, 4, LeafPayload(0.7, np.linspace(-1, 1, 12)),
                    max_depth=3)
    o, d = ray_set(52, 24)
    render_case("b4_single_leaf", t, o, d, 53, 0.3)

    # --- calibrate cases ----------------------------------------------------------
    rng = np.random.default_rng(100)
    t = irregular_tree(101, depth=3, basis_count=1, splits=10, merges=3, resplits=3, max_depth=5)
    acc = np.zeros(t.capacity); acc[t.leaf_ids()] = rng.uniform(0.0, 5.0, t.leaf_count)
    calib_case("recursive", t, acc, 4.6, 0.1, True)
    t = irregular_tree(102, depth=3, basis_count=4, splits=10, merges=3, resplits=3, max_depth=5)
    acc = np.zeros(t.capacity)
    acc[t.leaf_ids()] = np.round(rng.uniform(0.0, 3.0, t.leaf_count), 1)  # many ties
    calib_case("oneshot_ties", t, acc, 2.6, 0.3, False)
    t = irregular_tree(103, depth=3, basis_count=1, splits=6, merges=2, resplits=2, max_depth=5)
    acc = np.zeros(t.capacity); acc[t.leaf_ids()] = rng.uniform(0.0, 5.0, t.leaf_count)
    calib_case("threshold", t, acc, 4.5, 0.0, False, threshold=4.0)
    t = irregular_tree(104, depth=3, basis_count=4, splits=6, merges=2, resplits=2, max_depth=5,
                       sigma_range=(0.0, 1.0))
    calib_case("sigma_target", t, np.zeros(t.capacity), 0.9, 0.05, True, target="sigma")
    t = irregular_tree(105, depth=3, basis_count=1, splits=4, merges=1, resplits=1, max_depth=4)
    o, d = ray_set(106, 300, specials=False)
    _, _, sig = render_and_backprop(t, o, d, np.zeros((o.shape[0], 3)), 0.0)
    calib_case("rendered", t, sig, 0.3, 0.02, True)
    t = irregular_tree(107, depth=2, basis_count=1, splits=12, merges=0, resplits=0, max_depth=3)
    acc = np.zeros(t.capacity); acc[t.leaf_ids()] = rng.uniform(0.5, 5.0, t.leaf_count)
    calib_case("capped_gamma1", t, acc, 0.0, 1.0, False)
    # merge-order stress: wide dynamic range payloads so summation order matters
    t = irregular_tree(108, depth=3, basis_count=16, splits=4, merges=1, resplits=1, max_depth=5)
    lv = t.leaf_ids()
    mag = 10.0 ** rng.integers(-12, 12, (lv.size, 48))
    t.sh[lv] = (rng.normal(0.0, 1.0, (lv.size, 48)) * mag).astype(np.float32)
    t.sigma[lv] = (rng.uniform(0.0, 1.0, lv.size) * 10.0 ** rng.integers(-12, 12, lv.size)).astype(np.float32)
    acc = np.zeros(t.capacity); acc[lv] = rng.uniform(0.0, 1.0, lv.size) * 10.0 ** rng.integers(-8, 0, lv.size)
    calib_case("merge_order", t, acc, 0.05, 0.05, True)

    remap_case()
    train_case()
    config1()


def remap_case():
    """RmsPropState.remap across a recursive calibrate (optim.py:89-104)."""
    from octrf.optim import RmsPropState
    from octrf.scene_io import _level_order
    rng = np.random.default_rng(500)
    t = irregular_tree(501, depth=3, basis_count=4, splits=8, merges=2, resplits=2, max_depth=5)
    out = dict(pool_arrays(t))
    lv = t.leaf_ids()
    acc = np.zeros(t.capacity)
    acc[lv] = np.where(rng.uniform(size=lv.size) < 0.985, 0.0, rng.uniform(0.0, 5.0, lv.size))
    state = RmsPropState(t)
    state.v_sigma[:] = rng.uniform(0.0, 1e-3, t.capacity)
    state.v_sh[:] = rng.uniform(0.0, 1e-3, state.v_sh.shape)
    out.update(acc=acc, v_sigma=state.v_sigma.copy(), v_sh=state.v_sh.copy())
    buf = SignalBuffer(t)
    buf.accumulator[:] = acc
    report = calibrate(t, buf, CalibrationConfig(tau=0.0, gamma=0.1, recursive=True))
    state.remap(report)
    order, _ = _level_order(t)
    is_leaf = t._leaf[order] == 1
    out.update(tau=np.float64(0.0), gamma=np.float64(0.1),
               rounds=np.int64(report.recursion_rounds), merges=np.int64(report.merges_applied),
               splits=np.int64(report.splits_applied),
               canon_is_leaf=is_leaf, canon_v_sigma=state.v_sigma[order],
               canon_v_sh=state.v_sh[order])
    np.savez_compressed(os.path.join(HERE, "optim_remap.npz"), **out)
    print("remap", report.to_json())


class _Bundle:
    def __init__(self, origins, dirs, targets):
        self.origins, self.dirs, self.targets, self.heldout = origins, dirs, targets, []


def train_case():
    """A short train() run (optim.py:169-195): loss per epoch and leaf counts."""
    from octrf.optim import TrainConfig, train
    from octrf.sh import sh_from_rgb
    sh_in = sh_from_rgb(np.array([0.8, 0.3, 0.2]), 1)

    def ball(c):
        inside = np.linalg.norm(c, axis=1) <= 0.55
        return np.where(inside, 8.0, 0.0), np.where(inside[:, None], sh_in, 0.0)

    truth = build_dense(3, (0.0, 0.0, 0.0), 1.0, 1, ball, max_depth=5)
    o, d = ray_set(601, 2000, specials=False, miss_fraction=0.05)
    targets = render_rays(truth, o, d, 1.0, early_stop_eps=0.0)
    trainee = build_dense(2, (0.0, 0.0, 0.0), 1.0, 1, LeafPayload(0.3, [0.0, 0.0, 0.0]), max_depth=5)
    cfg = TrainConfig(epochs=6, interval=2, tau=0.5, gamma=0.1, batch_size=500, seed=3)
    _, hist = train(trainee, _Bundle(o, d, targets), cfg)
    out = dict(origins=o, dirs=d, targets=targets,
               loss=np.array([h["loss"] for h in hist]),
               leaf_count=np.array([h["leaf_count"] for h in hist]),
               final_dot1=np.frombuffer(dot1_bytes(trainee), dtype=np.uint8))
    np.savez_compressed(os.path.join(HERE, "train_small.npz"), **out)
    print("train", [round(h["loss"], 6) for h in hist], [h["leaf_count"] for h in hist])


class _HeldoutBundle(_Bundle):
    def __init__(self, origins, dirs, targets, heldout):
        super().__init__(origins, dirs, targets)
        self.heldout = heldout


def train_heldout_case():
    """train() with held-out views (optim.py:157-195): the per-epoch history
    including heldout_psnr (render_image of each held-out camera vs its
    image, metrics.psnr), and the held-out PSNR of the final tree."""
    from octrf.optim import TrainConfig, heldout_psnr, train
    from octrf.render import render_image
    from octrf.sh import sh_from_rgb
    sh_in = sh_from_rgb(np.array([0.2, 0.7, 0.4]), 4)

    def ball(c):
        inside = np.linalg.norm(c - np.array([0.1, -0.05, 0.0]), axis=1) <= 0.5
        return np.where(inside, 6.0, 0.0), np.where(inside[:, None], sh_in, 0.0)

    truth = build_dense(3, (0.0, 0.0, 0.0), 1.0, 4, ball, max_depth=5)
    o, d = ray_set(701, 3000, specials=False, miss_fraction=0.05)
    targets = render_rays(truth, o, d, 1.0, early_stop_eps=0.0)
    f = scenes.focal_from_angle(24, scenes.FOV_40)
    cams = [Camera(24, 20, f, scenes.orbit_pose(3.5, az, el)) for az, el in ((0.3, 0.4), (2.2, -0.2))]
    heldout = [(c, render_image(truth, c, 1.0)) for c in cams]
    trainee = build_dense(2, (0.0, 0.0, 0.0), 1.0, 4, LeafPayload(0.3, [0.0] * 12), max_depth=5)
    cfg = TrainConfig(epochs=4, interval=2, tau=0.3, gamma=0.1, batch_size=600, seed=5)
    _, hist = train(trainee, _HeldoutBundle(o, d, targets, heldout), cfg)
    out = dict(origins=o, dirs=d, targets=targets,
               cam_w=np.array([c.width for c in cams]), cam_h=np.array([c.height for c in cams]),
               cam_f=np.array([c.focal for c in cams]), cam_pose=np.stack([c.cam_to_world for c in cams]),
               heldout_images=np.stack([im for _, im in heldout]),
               loss=np.array([h["loss"] for h in hist]), psnr=np.array([h["psnr"] for h in hist]),
               leaf_count=np.array([h["leaf_count"] for h in hist]),
               final_psnr=np.float64(heldout_psnr(trainee, _HeldoutBundle(o, d, targets, heldout), 1.0)),
               final_dot1=np.frombuffer(dot1_bytes(trainee), dtype=np.uint8))
    np.savez_compressed(os.path.join(HERE, "train_heldout.npz"), **out)
    print("train_heldout", [round(h["psnr"], 4) for h in hist], [h["leaf_count"] for h in hist])


if __name__ == "__main__":
    if sys.argv[1:] == ["train_heldout"]:
        train_heldout_case()
    else:
        main()
