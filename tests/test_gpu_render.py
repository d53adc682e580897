"""GPU parity of traversal, forward and backward against the reference.

Two checkers: the golden fixtures (outputs of the reference itself, see
tests/golden/make_golden.py) and the C oracle (oracle/dot_oracle.c) on
fresh seeded inputs.  Bars (BASELINE.json north_star): leaf ids, t_entry and
delta bit-exact; rgb / T_final / weight sum / loss / gradients / signal within
1e-4 abs + 1e-3 rel (the CUDA path shades in fp32, accumulates in fp64).
"""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN

from helpers import assert_grads_close  # noqa: E402

pytestmark = pytest.mark.gpu

ATOL, RTOL = 1e-4, 1e-3
RENDER_CASES = sorted(glob.glob(os.path.join(GOLDEN, "render_*.npz")))


def _tree(z):
    from paper_2307_15333_b200.octree import from_pool_arrays
    return from_pool_arrays(z, device="cuda")


@pytest.fixture(params=RENDER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
def case(request):
    return np.load(request.param)


def test_segments_bit_exact(case):
    from paper_2307_15333_b200.render import segment_batch
    tree = _tree(case)
    off, leaf, t, d = segment_batch(tree, case["origins"], case["dirs"], float(case["t_near"]),
                                    float(case["t_far"]))
    np.testing.assert_array_equal(off, case["seg_offsets"])
    np.testing.assert_array_equal(leaf, case["seg_leaf"])
    np.testing.assert_array_equal(t, case["seg_t"])
    np.testing.assert_array_equal(d, case["seg_delta"])


@pytest.mark.parametrize("tag,eps", [("eps", 1e-4), ("noeps", 0.0)])
def test_forward_matches_reference(case, tag, eps):
    from paper_2307_15333_b200.render import render_rays
    tree = _tree(case)
    rgb, tfin, wsum = render_rays(tree, case["origins"], case["dirs"], case["bg"], eps,
                                  float(case["t_near"]), float(case["t_far"]), return_aux=True)
    np.testing.assert_allclose(rgb, case[f"rgb_{tag}"], atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(tfin, case[f"tfin_{tag}"], atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(wsum, case[f"wsum_{tag}"], atol=ATOL, rtol=RTOL)


@pytest.mark.parametrize("tag,eps", [("eps", 1e-4), ("noeps", 0.0)])
def test_backward_matches_reference(case, tag, eps):
    from paper_2307_15333_b200.render import render_and_backprop
    tree = _tree(case)
    loss, grads, signal = render_and_backprop(tree, case["origins"], case["dirs"], case["targets"],
                                              case["bg"], eps, float(case["t_near"]),
                                              float(case["t_far"]))
    assert loss == pytest.approx(float(case[f"loss_{tag}"]), rel=RTOL, abs=ATOL)
    assert_grads_close(grads.dsigma, case[f"dsigma_{tag}"], what="dsigma")
    assert_grads_close(grads.dsh, case[f"dsh_{tag}"], what="dsh")
    np.testing.assert_array_equal(grads.touched, case[f"touched_{tag}"])
    np.testing.assert_allclose(signal, case[f"signal_{tag}"], atol=ATOL, rtol=RTOL)


def test_config1_golden():
    """BASELINE.json configs[0] end to end against the reference's outputs."""
    from paper_2307_15333_b200.render import render_and_backprop, render_rays, segment_batch
    from paper_2307_15333_b200.scene_io import load_tree_bytes
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    tree = load_tree_bytes(z["scene_dot1"].tobytes(), device="cuda")
    off, leaf, t, d = segment_batch(tree, z["origins"], z["dirs"])
    np.testing.assert_array_equal(off, z["seg_offsets"])
    np.testing.assert_array_equal(leaf, z["seg_leaf"])
    np.testing.assert_array_equal(t, z["seg_t"])
    np.testing.assert_array_equal(d, z["seg_delta"])
    rgb, tfin, wsum = render_rays(tree, z["origins"], z["dirs"], 1.0, return_aux=True)
    np.testing.assert_allclose(rgb, z["rgb"], atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(tfin, z["tfin"], atol=ATOL, rtol=RTOL)
    loss, grads, signal = render_and_backprop(tree, z["origins"], z["dirs"], z["targets"], 1.0)
    assert loss == pytest.approx(float(z["loss"]), rel=RTOL, abs=ATOL)
    np.testing.assert_array_equal(grads.touched, z["touched"])
    assert_grads_close(grads.dsigma[z["touched"]], z["dsigma_touched"], what="dsigma")
    assert_grads_close(grads.dsh[z["touched"]], z["dsh_touched"], what="dsh")
    np.testing.assert_allclose(signal, z["signal"], atol=ATOL, rtol=RTOL)


@pytest.mark.parametrize("B", [1, 4, 9, 16])
def test_random_trees_vs_oracle(oracle, B):
    """Fresh seeded irregular trees (non-canonical pools) through the C oracle."""
    from paper_2307_15333_b200.render import render_and_backprop, render_rays, segment_batch
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(700 + B, B, depth=3, splits=20, merges=5, max_depth=5, device="cuda")
    o, d = ray_batch(800 + B, 3000)
    tg = np.random.default_rng(B).uniform(0, 1, (o.shape[0], 3))
    ref = oracle.segment_batch(tree, o, d)
    got = segment_batch(tree, o, d)
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)
    for eps in (1e-4, 0.0):
        rgb, tf, ws = render_rays(tree, o, d, (0.1, 0.5, 0.9), eps, return_aux=True)
        r_rgb, r_tf, r_ws = oracle.render_rays(tree, o, d, (0.1, 0.5, 0.9), eps, return_aux=True)
        np.testing.assert_allclose(rgb, r_rgb, atol=ATOL, rtol=RTOL)
        np.testing.assert_allclose(tf, r_tf, atol=ATOL, rtol=RTOL)
        np.testing.assert_allclose(ws, r_ws, atol=ATOL, rtol=RTOL)
        loss, g, sig = render_and_backprop(tree, o, d, tg, 0.3, eps)
        r_loss, r_g, r_sig = oracle.render_and_backprop(tree, o, d, tg, 0.3, eps)
        assert loss == pytest.approx(r_loss, rel=RTOL, abs=ATOL)
        assert_grads_close(g.dsigma, r_g.dsigma, what="dsigma")
        assert_grads_close(g.dsh, r_g.dsh, what="dsh")
        np.testing.assert_array_equal(g.touched, r_g.touched)
        np.testing.assert_allclose(sig, r_sig, atol=ATOL, rtol=RTOL)


def test_depth_definition(oracle):
    from paper_2307_15333_b200.render import render_rays
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(901, 4, depth=2, splits=10, merges=2, max_depth=4, device="cuda")
    o, d = ray_batch(902, 500)
    _, depth = render_rays(tree, o, d, 1.0, return_depth=True)
    np.testing.assert_allclose(depth, oracle.render_depth(tree, o, d), atol=ATOL, rtol=RTOL)


def test_empty_and_miss_batches():
    from paper_2307_15333_b200.render import render_and_backprop, render_rays
    from helpers import irregular_tree
    tree = irregular_tree(5, 1, depth=1, splits=0, merges=0, max_depth=3, device="cuda")
    empty = np.zeros((0, 3))
    assert render_rays(tree, empty, empty, 1.0).shape == (0, 3)
    loss, g, sig = render_and_backprop(tree, empty, empty, empty, 1.0)
    assert loss == 0.0 and g.touched.size == 0 and not sig.any()
    o = np.array([[0.0, 0.0, 5.0], [0.0, 5.0, 0.0]])
    d = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    tg = np.array([[1.0, 1.0, 1.0], [0.0, 0.0, 0.0]])
    loss, g, sig = render_and_backprop(tree, o, d, tg, 1.0, early_stop_eps=0.0)
    assert loss == pytest.approx(1.5)
    assert g.touched.size == 0 and not g.dsigma.any() and not sig.any()


@pytest.mark.parametrize("size", [(64, 64), (37, 23)])
def test_camera_render_in_kernel_rays(oracle, size):
    """render_image with in-kernel camera rays (8x4 warp tiles, odd image sizes)
    vs the reference path on camera.rays() through the oracle."""
    from paper_2307_15333_b200 import scenes
    from paper_2307_15333_b200.render import render_image, render_view
    from paper_2307_15333_b200.scene_io import Camera, load_tree_bytes
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    tree = load_tree_bytes(z["scene_dot1"].tobytes(), device="cuda")
    W, H = size
    cam = Camera(W, H, scenes.focal_from_angle(W, scenes.FOV_40),
                 scenes.orbit_pose(**scenes.CONFIG1_POSE))
    img = render_image(tree, cam, 1.0, exact_rays=False)
    o, d = cam.rays()
    want = oracle.render_rays(tree, o, d, 1.0).reshape(H, W, 3)
    np.testing.assert_allclose(img, want, atol=ATOL, rtol=RTOL)
    exact = render_image(tree, cam, 1.0)
    np.testing.assert_allclose(exact, want, atol=ATOL, rtol=RTOL)
    rgb, tfin, depth = render_view(tree, cam, 1.0, return_aux=True)
    assert rgb.shape == (H, W, 3) and tfin.shape == (H, W)
    np.testing.assert_allclose(depth.cpu().numpy().reshape(-1), oracle.render_depth(tree, o, d),
                               atol=ATOL, rtol=RTOL)


def test_length_mismatch_raises():
    from paper_2307_15333_b200.errors import InputError
    from paper_2307_15333_b200.render import render_and_backprop
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(6, 1, depth=1, splits=0, merges=0, max_depth=3, device="cuda")
    o, d = ray_batch(7, 4)
    with pytest.raises(InputError):
        render_and_backprop(tree, o, d, np.zeros((3, 3)), 0.0)


def test_device_exp_ref(oracle):
    """Every alpha = exp(-sigma delta) on the device uses exp_ref, which must
    equal glibc's exp (the reference's) bit for bit."""
    import torch
    from paper_2307_15333_b200 import _lib
    from test_host import _exp_args
    x = _exp_args(1 << 20, seed=3)
    want = oracle.exp(x)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    _lib.call("dot_exp_ref_device", _lib.ptr(xd), _lib.ptr(yd), x.size, _lib.stream_ptr())
    got = yd.cpu().numpy()
    same = got.view(np.uint64) == want.view(np.uint64)
    assert np.all(same | (np.isnan(got) & np.isnan(want))), x[~same][:5]


def test_ray_index_reads_in_place():
    """render_and_backprop(ray_index=...) == the same call on the gathered
    batch (atomic path within fp32-atomic noise; deterministic path bit for
    bit, including the reduction order)."""
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import render_and_backprop
    tree = irregular_tree(21, 9, depth=3, splits=60, max_depth=6, device="cuda")
    o, d = ray_batch(22, 60000)
    t = np.random.default_rng(23).uniform(0, 1, (o.shape[0], 3))
    o, d, t = (torch.from_numpy(x).cuda() for x in (o, d, t))
    idx = torch.randperm(o.shape[0], generator=torch.Generator().manual_seed(1))[:40000].cuda()
    l1, g1, s1 = render_and_backprop(tree, o[idx], d[idx], t[idx], 0.2)
    g1 = (g1.dsigma.clone(), g1.dsh.clone(), g1.touched_mask.clone())
    s1 = s1.clone()
    l2, g2, s2 = render_and_backprop(tree, o, d, t, 0.2, ray_index=idx)
    assert float(l2) == pytest.approx(float(l1), rel=1e-9)
    torch.testing.assert_close(g2.dsigma, g1[0], atol=1e-6, rtol=1e-4)
    torch.testing.assert_close(g2.dsh, g1[1], atol=1e-6, rtol=1e-4)
    assert torch.equal(g2.touched_mask, g1[2])
    torch.testing.assert_close(s2, s1, atol=1e-12, rtol=1e-12)
    _, h1, r1 = render_and_backprop(tree, o[idx], d[idx], t[idx], 0.2, deterministic=True)
    h1 = (h1.dsigma.clone(), h1.dsh.clone())
    r1 = r1.clone()
    _, h2, r2 = render_and_backprop(tree, o, d, t, 0.2, ray_index=idx, deterministic=True)
    assert torch.equal(h2.dsigma, h1[0]) and torch.equal(h2.dsh, h1[1]) and torch.equal(r2, r1)


def test_long_rays_resume_past_the_record_buffer(oracle):
    """Rays with more composited segments than the backward's per-ray record
    buffer (128) resume their walk in pass 2: a dense depth-6 tree, eps = 0
    and low density make diagonal rays composite ~190 segments."""
    from paper_2307_15333_b200.octree import build_dense
    from paper_2307_15333_b200.render import render_and_backprop
    rng = np.random.default_rng(5)

    def init(c):
        return rng.uniform(0.0, 0.3, len(c)), rng.normal(0.0, 0.5, (len(c), 3))

    tree = build_dense(6, (0.0, 0.0, 0.0), 1.0, 1, init, max_depth=6, device="cuda")
    n = 600
    o = np.tile([-1.5, -1.4, -1.3], (n, 1)) + rng.uniform(-0.2, 0.2, (n, 3))
    d = np.ones((n, 3)) + rng.uniform(-0.05, 0.05, (n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tg = rng.uniform(0, 1, (n, 3))
    r_off, _, _, _ = oracle.segment_batch(tree, o, d)
    assert np.diff(r_off).max() > 160
    for det in (False, True):
        loss, g, sig = render_and_backprop(tree, o, d, tg, 0.5, 0.0, deterministic=det)
        r_loss, r_g, r_sig = oracle.render_and_backprop(tree, o, d, tg, 0.5, 0.0)
        assert loss == pytest.approx(r_loss, rel=RTOL, abs=ATOL)
        assert_grads_close(g.dsigma, r_g.dsigma, what="dsigma")
        assert_grads_close(g.dsh, r_g.dsh, what="dsh")
        np.testing.assert_array_equal(g.touched, r_g.touched)
        np.testing.assert_allclose(sig, r_sig, atol=ATOL, rtol=RTOL)


def test_render_views_equals_per_view():
    """render_views (all views in one launch) == render_view per camera, bit
    for bit (same per-pixel code)."""
    import torch
    from paper_2307_15333_b200 import scenes
    from paper_2307_15333_b200.render import render_view, render_views
    from paper_2307_15333_b200.scene_io import Camera
    from helpers import irregular_tree
    tree = irregular_tree(8, 9, depth=3, splits=40, max_depth=6, device="cuda")
    focal, poses = scenes.hemisphere_cameras(5, 96, 72, 4.0, seed=2)
    cams = [Camera(96, 72, focal * (1.0 + 0.1 * i), p) for i, p in enumerate(poses)]
    rgb, tf, dep = render_views(tree, cams, (0.2, 0.3, 0.4), return_aux=True)
    for i, c in enumerate(cams):
        r1, t1, d1 = render_view(tree, c, (0.2, 0.3, 0.4), return_aux=True)
        assert torch.equal(rgb[i], r1) and torch.equal(tf[i], t1) and torch.equal(dep[i], d1)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 1 << 16, (1 << 20) + 5, 3 << 20])
def test_sched_order_is_a_permutation(n):
    """dot_sched_order must launch every warp exactly once whatever the table
    holds (a duplicate or missing warp would silently drop rays)."""
    import torch
    from paper_2307_15333_b200 import _lib
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    keys = torch.sort(torch.randint(0, 2 ** 31 - 1, (n,), generator=g, device="cuda", dtype=torch.int64)
                      .to(torch.int32)).values
    table = torch.randint(0, 3000, ((1 << 24) + (1 << 27),), generator=g, device="cuda",
                          dtype=torch.int64).to(torch.int16)
    nw = (n + 31) // 32
    order = torch.full((nw,), -1, dtype=torch.int32, device="cuda")
    _lib.call("dot_sched_order", _lib.ptr(keys), n, _lib.ptr(table), _lib.ptr(order), _lib.stream_ptr())
    assert torch.equal(torch.sort(order.to(torch.int64)).values, torch.arange(nw, device="cuda"))


def test_plan_sort_and_pool_keys():
    """dot_plan_sort is a stable key sort carrying the ray index (== torch's
    stable sort + gather), and a plan from precomputed pool keys equals the
    plan computed from the rays; the schedule is a permutation of the warps."""
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import plan_batch, pool_keys
    tree = irregular_tree(31, 4, depth=2, splits=10, max_depth=4, device="cuda")
    o, d = ray_batch(32, 50000)
    o, d = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    idx = torch.randperm(50000, generator=g, device="cuda")[:40000]
    p1 = plan_batch(tree, o, d, idx)
    keys = pool_keys(tree, o, d)
    p2 = plan_batch(tree, o, d, idx, keys=keys)
    ks, perm = torch.sort(keys[idx], stable=True)
    assert torch.equal(p1.sorted_keys, ks) and torch.equal(p2.sorted_keys, ks)
    assert torch.equal(p1.idx, idx[perm]) and torch.equal(p2.idx, idx[perm])
    nw = (40000 + 31) // 32
    for p in (p1, p2):
        assert torch.equal(torch.sort(p.warp_order.to(torch.int64)).values, torch.arange(nw, device="cuda"))


def _plan_ranked(rank, order, idx, ws=None, n_pool=None):
    import torch
    from paper_2307_15333_b200 import _lib
    n_pool, n = (rank.shape[0] if n_pool is None else n_pool), idx.shape[0]
    mode = 1 if order is not None else 0
    need = _lib.load().dot_plan_ranked_workspace(n_pool, n, mode)
    if ws is None or ws.numel() < need:
        ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    out = torch.full((n,), -7, dtype=torch.int64, device="cuda")
    _lib.call("dot_plan_ranked", _lib.ptr(rank), _lib.ptr(order), n_pool, _lib.ptr(idx), n, mode, None, 1, None,
              _lib.ptr(ws), ws.numel(), _lib.ptr(out), _lib.stream_ptr())
    return out, ws


def _a256(b):
    return (b + 255) // 256 * 256


def _plan_scratch_clear(ws, n_pool, n):
    """The regions of a plan workspace that must be zero between calls
    (bitmap + slack, claim bitmap, counters, cost histogram) are zero
    (plan.cu carve(): they precede the per-batch scratch)."""
    words = (n_pool + 31) // 32
    at_claim = _a256(4 * (words + 512))
    at_ctr = at_claim + _a256(4 * words) + _a256(4 * 4096)
    at_hist = at_ctr + 256
    return (not bool(ws[:at_claim].any()) and not bool(ws[at_claim:at_claim + 4 * words].any())
            and not bool(ws[at_ctr:at_ctr + 16].any()) and not bool(ws[at_hist:at_hist + 4096].any()))


def _cost_bucket(c):
    """plan.cu cost_bucket: three log-scale buckets per octave of cost + 1."""
    import torch
    x = c + 1
    m = torch.floor(torch.log2(x.double())).long()
    m = torch.where((1 << (m + 1)) <= x, m + 1, m)  # exact floor(log2) for integers
    m = torch.where((1 << m) > x, m - 1, m)
    return 3 * m + ((3 * x) >> m) - 3


def _regrouped(key_ordered, cost_of, window=128):
    """The plan's output with a cost column: inside each window of 128 slots
    the key-ordered rays stably partitioned by cost bucket (costs capped at
    1023), costliest first."""
    import torch
    bucket = _cost_bucket(torch.clamp(cost_of(key_ordered).long(), max=1023))
    out = key_ordered.clone()
    for b in range(0, key_ordered.numel(), window):
        order = torch.sort(-bucket[b:b + window], stable=True).indices
        out[b:b + window] = key_ordered[b:b + window][order]
    return out


def _check_warp_order(order, costs_of_slots, n, chunk):
    """A permutation of the warps; full chunks by non-increasing max cost
    (capped at 1023), a short last chunk last."""
    nw = (n + 31) // 32
    od = order.cpu().numpy()
    assert np.array_equal(np.sort(od), np.arange(nw))
    pad = np.zeros(nw * 32, dtype=np.int64)
    pad[:n] = costs_of_slots
    wc = np.minimum(pad.reshape(nw, 32).max(1), 1023)
    nfull = nw // chunk
    cc = wc[: nfull * chunk].reshape(nfull, chunk).max(1)
    firsts = od[: nfull * chunk: chunk]
    assert np.all(firsts % chunk == 0)
    for k in range(chunk):  # chunks stay contiguous
        assert np.array_equal(od[k: nfull * chunk: chunk], firsts + k)
    assert np.all(np.diff(cc[firsts // chunk]) <= 0)
    assert np.array_equal(od[nfull * chunk:], np.arange(nfull * chunk, nw))


def test_plan_ranked_warp_order():
    """dot_plan_ranked's fused warp order (warp costs gathered while placing)
    is the cost-ordered launch of dot_sched_order_costs for the same plan,
    for chunk 1 and 16, with a short last warp / chunk; its warp-cost
    scratch is left zeroed."""
    import torch
    from paper_2307_15333_b200 import _lib
    g = torch.Generator(device="cuda")
    g.manual_seed(12)
    n_pool = 400_003
    order = torch.randperm(n_pool, generator=g, device="cuda").to(torch.int32)
    rank = torch.empty(n_pool, dtype=torch.int32, device="cuda")
    rank[order.long()] = torch.arange(n_pool, dtype=torch.int32, device="cuda")
    costs = torch.randint(0, 1400, (n_pool,), generator=g, device="cuda").to(torch.int16)
    for n, chunk in ((70_001, 1), (70_001, 16), (65_536, 16), (333, 1)):
        for ordr in (order, None):
            idx = torch.randperm(n_pool, generator=g, device="cuda")[:n]
            mode = 1 if ordr is not None else 0
            need = _lib.load().dot_plan_ranked_workspace(n_pool, n, mode)
            ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
            out = torch.empty(n, dtype=torch.int64, device="cuda")
            wo = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")
            keyed = torch.sort(rank[idx].long()).values
            if ordr is not None:
                keyed = ordr[keyed].long()
            want = _regrouped(keyed, lambda v: costs[v])
            for rep in range(2):  # the second call on the returned workspace
                _lib.call("dot_plan_ranked", _lib.ptr(rank), _lib.ptr(ordr), n_pool, _lib.ptr(idx), n, mode,
                          _lib.ptr(costs), chunk, _lib.ptr(wo), _lib.ptr(ws), ws.numel(), _lib.ptr(out),
                          _lib.stream_ptr())
                torch.cuda.synchronize()
                assert torch.equal(out, want), "not the key order regrouped by cost in 128-ray windows"
                _check_warp_order(wo, costs[out].long().cpu().numpy(), n, chunk)
                assert _plan_scratch_clear(ws, n_pool, n), "scratch not left zeroed"
    # slots of a staged batch: ids name its rays in the ranked dataset, the
    # warp costs come per slot (above 2^21 rays the slot no longer packs
    # with its cost into the tag: the cost is gathered by slot instead)
    big = 1 << 21
    n_pool_b = big + 5000
    order_b = torch.randperm(n_pool_b, generator=g, device="cuda").to(torch.int32)
    rank_b = torch.empty(n_pool_b, dtype=torch.int32, device="cuda")
    rank_b[order_b.long()] = torch.arange(n_pool_b, dtype=torch.int32, device="cuda")
    for n in (big, big + 1000):
        ids = torch.randperm(n_pool_b, generator=g, device="cuda")[:n]
        slot_cost = torch.randint(0, 1400, (n,), generator=g, device="cuda").to(torch.int16)
        ws = torch.zeros(_lib.load().dot_plan_ranked_workspace(n_pool_b, n, 2), dtype=torch.uint8, device="cuda")
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        wo = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        _lib.call("dot_plan_ranked", _lib.ptr(rank_b), None, n_pool_b, _lib.ptr(ids), n, 2, _lib.ptr(slot_cost), 16,
                  _lib.ptr(wo), _lib.ptr(ws), ws.numel(), _lib.ptr(out), _lib.stream_ptr())
        torch.cuda.synchronize()
        assert torch.equal(out, _regrouped(torch.sort(rank_b[ids].long()).indices, lambda v: slot_cost[v]))
        _check_warp_order(wo, slot_cost[out].long().cpu().numpy(), n, 16)
    for n in (1, 4097, 70_001):
        ids = torch.randperm(n_pool, generator=g, device="cuda")[:n]
        slot_cost = torch.randint(0, 1400, (n,), generator=g, device="cuda").to(torch.int16)
        need = _lib.load().dot_plan_ranked_workspace(n_pool, n, 2)
        ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        wo = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        _lib.call("dot_plan_ranked", _lib.ptr(rank), None, n_pool, _lib.ptr(ids), n, 2, _lib.ptr(slot_cost), 1,
                  _lib.ptr(wo), _lib.ptr(ws), ws.numel(), _lib.ptr(out), _lib.stream_ptr())
        torch.cuda.synchronize()
        assert torch.equal(out, _regrouped(torch.sort(rank[ids].long()).indices, lambda v: slot_cost[v]))
        _check_warp_order(wo, slot_cost[out].long().cpu().numpy(), n, 1)
        assert _plan_scratch_clear(ws, n_pool, n)
    # one workspace sized for the largest batch serves smaller ones (the
    # last batch of an epoch): the zero regions do not move with n
    need = _lib.load().dot_plan_ranked_workspace(n_pool, 70_001, 0)
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    for n in (70_001, 50_000, 70_001, 333, 12_345):
        idx = torch.randperm(n_pool, generator=g, device="cuda")[:n]
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        wo = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        _lib.call("dot_plan_ranked", _lib.ptr(rank), None, n_pool, _lib.ptr(idx), n, 0, _lib.ptr(costs), 1,
                  _lib.ptr(wo), _lib.ptr(ws), ws.numel(), _lib.ptr(out), _lib.stream_ptr())
        torch.cuda.synchronize()
        assert torch.equal(out, _regrouped(torch.sort(rank[idx].long()).values, lambda v: costs[v]))
        _check_warp_order(wo, costs[out].long().cpu().numpy(), n, 1)
        assert _plan_scratch_clear(ws, n_pool, n)
    # repeats and invalid indices with a cost column: still a permutation of
    # the batch (the appended rays are regrouped like the placed ones) and a
    # valid launch order; the workspace stays reusable
    for mode in (0, 1, 2):
        base = torch.randperm(n_pool, generator=g, device="cuda")[:5000]
        idx = torch.cat([base, base[:700], torch.tensor([-5, n_pool, n_pool + 7], device="cuda")])
        idx = idx[torch.randperm(idx.shape[0], generator=g, device="cuda")]
        n = idx.shape[0]
        cst = slot_cost if mode == 2 else costs
        if mode == 2:
            cst = torch.randint(0, 1400, (n,), generator=g, device="cuda").to(torch.int16)
        need = _lib.load().dot_plan_ranked_workspace(n_pool, n, mode)
        ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        wo = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        for rep in range(2):
            _lib.call("dot_plan_ranked", _lib.ptr(rank), _lib.ptr(order if mode == 1 else None), n_pool, _lib.ptr(idx),
                      n, mode, _lib.ptr(cst), 1, _lib.ptr(wo), _lib.ptr(ws), ws.numel(), _lib.ptr(out),
                      _lib.stream_ptr())
            torch.cuda.synchronize()
            if mode == 2:  # slots: a permutation of 0..n-1
                assert torch.equal(torch.sort(out).values, torch.arange(n, device="cuda"))
                slot_costs = cst[out].long()
            else:
                # positions: valid ids come back as rank[id]; pool rays: as
                # order[rank[id]] == id; invalid indices as they were
                ok = (idx >= 0) & (idx < n_pool)
                want = torch.where(ok, rank[idx.clamp(0, n_pool - 1)].long(), idx) if mode == 0 else idx
                assert torch.equal(torch.sort(out).values, torch.sort(want).values)
                valid = (out >= 0) & (out < n_pool)
                slot_costs = torch.where(valid, cst[out.clamp(0, n_pool - 1)].long(), torch.zeros_like(out))
            _check_warp_order(wo, slot_costs.cpu().numpy(), n, 1)
            assert _plan_scratch_clear(ws, n_pool, n)
    # bad arguments are refused
    from paper_2307_15333_b200.errors import InputError
    with pytest.raises(InputError):
        _lib.call("dot_plan_ranked", _lib.ptr(rank), None, n_pool, _lib.ptr(ids), n, 1, None, 1, None,
                  _lib.ptr(ws), ws.numel(), _lib.ptr(out), _lib.stream_ptr())  # POOL_RAYS without order
    with pytest.raises(InputError):
        _lib.call("dot_plan_ranked", _lib.ptr(rank), None, n_pool, _lib.ptr(ids), n, 2, None, 1, None,
                  _lib.ptr(ws), 64, _lib.ptr(out), _lib.stream_ptr())  # workspace too small


def test_plan_ranked_counting_sort():
    """dot_plan_ranked puts a batch of distinct pool rays in rank order
    (== order[sort(rank[batch])]) for pools that are not a multiple of the
    bitmap word / block, reuses its workspace (left zeroed), and with
    repeated or out-of-range indices still returns a permutation of the
    batch: the placed rays in rank order, the rest after them."""
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    for n_pool, n in ((1, 1), (37, 20), (65536 + 33, 4097), (300_001, 65_536), (2_000_000, 1 << 20)):
        order = torch.randperm(n_pool, generator=g, device="cuda").to(torch.int32)
        rank = torch.empty(n_pool, dtype=torch.int32, device="cuda")
        rank[order.long()] = torch.arange(n_pool, dtype=torch.int32, device="cuda")
        ws = None
        for rep in range(2):
            idx = torch.randperm(n_pool, generator=g, device="cuda")[:n]
            out, ws = _plan_ranked(rank, order, idx, ws)
            want = order[torch.sort(rank[idx].long()).values].long()
            assert torch.equal(out, want), (n_pool, n, rep)
            # the pool stored in key order: positions out (order NULL), and
            # positions in as well (rank NULL)
            out, ws = _plan_ranked(rank, None, idx, ws)
            assert torch.equal(out, torch.sort(rank[idx].long()).values)
            out, ws = _plan_ranked(None, None, idx, ws, n_pool=n_pool)
            assert torch.equal(out, torch.sort(idx).values)
            torch.cuda.synchronize()
            assert _plan_scratch_clear(ws, n_pool, n), "bitmap not cleared"
    # repeats and invalid indices
    n_pool = 5000
    order = torch.randperm(n_pool, generator=g, device="cuda").to(torch.int32)
    rank = torch.empty(n_pool, dtype=torch.int32, device="cuda")
    rank[order.long()] = torch.arange(n_pool, dtype=torch.int32, device="cuda")
    base = torch.randperm(n_pool, generator=g, device="cuda")[:3000]
    idx = torch.cat([base, base[:500], torch.tensor([-1, n_pool, 1 << 40], device="cuda")])
    idx = idx[torch.randperm(idx.shape[0], generator=g, device="cuda")]
    out, _ = _plan_ranked(rank, order, idx)
    assert torch.equal(torch.sort(out).values, torch.sort(idx).values)
    placed = out[:3000]
    assert torch.equal(placed, order[torch.sort(rank[base].long()).values].long())


def test_pool_rank_plans_match_sorted_plans():
    """pool_rank's rank / order are inverse permutations in 62-bit key
    order; a plan_batch(rank=) plan is a permutation of the batch in key
    order and gives the same loss / gradients / signal as a sorted plan."""
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200 import _lib
    from paper_2307_15333_b200.render import (BackpropWorkspace, PoolRank, plan_batch, pool_keys, pool_rank,
                                              ray_costs, render_and_backprop)
    from paper_2307_15333_b200.errors import InputError
    tree = irregular_tree(41, 16, depth=3, splits=40, merges=4, max_depth=6, device="cuda")
    o, d = ray_batch(42, 90_001)
    t = np.random.default_rng(43).uniform(0, 1, (o.shape[0], 3))
    o, d, t = (torch.from_numpy(x).cuda() for x in (o, d, t))
    pr = pool_rank(tree, o, d)
    n_pool = o.shape[0]
    assert torch.equal(pr.rank[pr.order.long()], torch.arange(n_pool, dtype=torch.int32, device="cuda"))
    keys = torch.empty(n_pool, dtype=torch.int64, device="cuda")
    view, _ = tree.tree_view()
    _lib.call("dot_ray_keys", _lib.ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), n_pool, _lib.ptr(keys),
              _lib.stream_ptr())
    assert bool((keys[pr.order.long()].diff() >= 0).all())
    g = torch.Generator(device="cuda")
    g.manual_seed(44)
    idx = torch.randperm(n_pool, generator=g, device="cuda")[:70_000]
    side = torch.cuda.Stream()
    costs = ray_costs(tree, o, d)
    results = []
    po, pd, pt, pc = pr.permute(o, d, t, costs)  # the pool stored in key order
    for kw in ({"keys": pool_keys(tree, o, d)}, {"rank": pr}, {"rank": pr, "costs": costs},
               {"rank": pr.in_key_order(), "costs": pc}, {"rank": PoolRank.identity(n_pool, "cuda"), "costs": pc}):
        permuted = kw.get("rank") is not None and kw["rank"].order is None
        oo, dd, tt = (po, pd, pt) if permuted else (o, d, t)
        # a rank maps caller ray ids; the identity rank takes key positions
        ii = pr.positions(idx) if permuted and kw["rank"].rank is None else idx
        p = plan_batch(tree, oo, dd, ii, stream=side, **kw)
        if "rank" in kw:
            p.wait()
            assert p.sorted_keys is None
            want = torch.sort(pr.rank[idx].long()).values
            keyed = want if permuted else pr.order[want].long()
            if "costs" in kw:  # regrouped by cost inside 128-ray windows
                keyed = _regrouped(keyed, lambda v: kw["costs"][v])
            assert torch.equal(p.idx, keyed)
            assert (p.warp_order is not None) == ("costs" in kw)
        ws = BackpropWorkspace.for_tree(tree)
        results.append(render_and_backprop(tree, oo, dd, tt, 0.5, ray_index=ii, workspace=ws, plan=p))
    (l0, g0, s0) = results[0]
    for (l1, g1, s1) in results[1:]:
        assert float(l1) == pytest.approx(float(l0), rel=1e-9)
        torch.testing.assert_close(g1.dsh, g0.dsh, atol=1e-7, rtol=1e-4)
        torch.testing.assert_close(g1.dsigma, g0.dsigma, atol=1e-7, rtol=1e-4)
        assert torch.equal(g1.touched_mask, g0.touched_mask)
        torch.testing.assert_close(s1, s0, rtol=1e-12, atol=1e-15)
    with pytest.raises(InputError):
        plan_batch(tree, o, d, None, rank=pr)
    with pytest.raises(InputError):
        plan_batch(tree, o[:100], d[:100], idx[:10] % 100, rank=pr)


def test_large_batch_with_schedule_vs_oracle(oracle):
    """A batch large enough for the coherence sort and the learned warp
    schedule (several steps, so the table is warm) against the oracle."""
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import render_and_backprop
    tree = irregular_tree(90, 4, depth=3, splits=60, merges=4, max_depth=6, device="cuda")
    o, d = ray_batch(91, 100_000)
    tg = np.random.default_rng(92).uniform(0, 1, (o.shape[0], 3))
    for _ in range(3):  # warm the cost table
        render_and_backprop(tree, torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda(),
                            torch.from_numpy(tg).cuda(), 0.4)
    loss, g, sig = render_and_backprop(tree, o, d, tg, 0.4)
    r_loss, r_g, r_sig = oracle.render_and_backprop(tree, o, d, tg, 0.4)
    assert loss == pytest.approx(r_loss, rel=RTOL, abs=ATOL)
    assert_grads_close(g.dsigma, r_g.dsigma, what="dsigma")
    assert_grads_close(g.dsh, r_g.dsh, what="dsh")
    np.testing.assert_array_equal(g.touched, r_g.touched)
    np.testing.assert_allclose(sig, r_sig, atol=ATOL, rtol=RTOL)


def test_pool_rank_misuse_is_refused():
    """PoolRank / plan_batch(rank=, ids=) argument errors raise InputError
    before any launch."""
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.errors import InputError
    from paper_2307_15333_b200.render import PoolRank, plan_batch, pool_keys, pool_rank
    tree = irregular_tree(3, 4, depth=2, splits=5, max_depth=4, device="cuda")
    o, d = ray_batch(4, 1000)
    o, d = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    pr = pool_rank(tree, o, d)
    idx = torch.arange(100, device="cuda")
    with pytest.raises(InputError):
        PoolRank(pr.rank.long(), pr.order)  # not int32
    with pytest.raises(InputError):
        PoolRank(pr.rank, pr.order[:10])  # lengths differ
    with pytest.raises(InputError):
        PoolRank.identity(1000, "cuda").permute(o)  # no order to permute by
    with pytest.raises(InputError):
        pool_rank(tree, o, d, bits=40)
    with pytest.raises(InputError):
        plan_batch(tree, o, d, idx, rank=pr, keys=pool_keys(tree, o, d))
    with pytest.raises(InputError):
        plan_batch(tree, o, d, idx, ids=idx)  # ids without a rank
    with pytest.raises(InputError):
        plan_batch(tree, o[:100], d[:100], None, rank=pr, ids=idx[:50])  # ids not one per row
    with pytest.raises(InputError):
        plan_batch(tree, o, d, idx, rank=pr, costs=torch.zeros(10, dtype=torch.int16, device="cuda"))
    with pytest.raises(InputError):
        plan_batch(tree, o, d, idx, rank=pr, out=(torch.empty(10, dtype=torch.int64, device="cuda"),
                                                  torch.empty(1, dtype=torch.int32, device="cuda")))
    # positions map through the rank
    assert torch.equal(pr.positions(idx), pr.rank[idx].long())
