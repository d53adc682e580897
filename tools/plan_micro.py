"""Micro-benchmark of the batch plan kernels (no tree needed): a 2^26-ray
pool, 2^20-ray batches of distinct random positions, random u16 costs.
Times dot_plan_ranked (identity rank, rank + order, with / without the fused
warp order) and the sorted-keys plan (gather + radix sort + cost order)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2307_15333_b200 import _lib  # noqa: E402


def main():
    dev = torch.device("cuda")
    n_pool, n = 1 << 26, 1 << 20
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    order = torch.randperm(n_pool, generator=g, device=dev).to(torch.int32)
    rank = torch.empty(n_pool, dtype=torch.int32, device=dev)
    rank[order.long()] = torch.arange(n_pool, dtype=torch.int32, device=dev)
    costs = torch.randint(0, 300, (n_pool,), generator=g, device=dev).to(torch.int16)
    keys = torch.randint(0, 1 << 31, (n_pool,), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
    batches = [torch.randperm(n_pool, generator=g, device=dev)[:n] for _ in range(8)]
    ws = torch.zeros(_lib.load().dot_plan_ranked_workspace(n_pool, n, 2), dtype=torch.uint8, device=dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    wo = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    s = _lib.stream_ptr()

    slot_cost = costs[:n].contiguous()

    def ranked(rk, od, with_order, mode=None):
        mode = (1 if od is not None else 0) if mode is None else mode

        def f(idx):
            _lib.call("dot_plan_ranked", _lib.ptr(rk), _lib.ptr(od), n_pool, _lib.ptr(idx), n, mode,
                      (_lib.ptr(slot_cost) if mode == 2 else _lib.ptr(costs)) if with_order else None, 1,
                      _lib.ptr(wo) if with_order else None, _lib.ptr(ws), ws.numel(), _lib.ptr(out), s)
        return f

    def sorted_keys(idx):
        k = torch.empty(n, dtype=torch.int32, device=dev)
        _lib.call("dot_gather_keys", _lib.ptr(keys), n_pool, _lib.ptr(idx), n, _lib.ptr(k), s)
        sk = torch.empty_like(k)
        _lib.call("dot_plan_sort", _lib.ptr(k), _lib.ptr(idx), n, 0, _lib.ptr(sk), _lib.ptr(out), s)
        _lib.call("dot_sched_order_costs", _lib.ptr(costs), n_pool, _lib.ptr(out), n, 1, _lib.ptr(wo), s)

    def cost_only(idx):
        _lib.call("dot_sched_order_costs", _lib.ptr(costs), n_pool, _lib.ptr(idx), n, 1, _lib.ptr(wo), s)

    cases = [("ranked identity", ranked(None, None, False)), ("ranked identity + order", ranked(None, None, True)),
             ("ranked rank+order", ranked(rank, order, False)),
             ("ranked rank+order + order", ranked(rank, order, True)),
             ("ranked slots + order", ranked(rank, None, True, mode=2)),
             ("sched_order_costs alone", cost_only), ("keys: gather+sort+cost order", sorted_keys)]
    for name, f in cases:
        for b in batches[:2]:
            f(b)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for r in range(3):
            for b in batches:
                f(b)
        e.record()
        torch.cuda.synchronize()
        print(f"{name:32s} {1000 * a.elapsed_time(e) / 24:8.1f} us")


if __name__ == "__main__":
    main()
