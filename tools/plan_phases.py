"""Phase timeline of the cooperative plan kernel (diagnostic build:
DOT_LIB_PATH=tools/variants/lib_diag.so): %globaltimer after each grid sync,
alone and beside a bandwidth-bound copy on another stream (the optimizer's
stand-in).  Phases: A mark, B count, C warp bases (+ repeats), D place
(+ gathers, appended rays), W cost regrouping, E chunk costs + histogram,
F bin scan, G scatter + clear."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2307_15333_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    dev = torch.device("cuda")
    n_pool, n = 1 << 26, 1 << 20
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    order = torch.randperm(n_pool, generator=g, device=dev).to(torch.int32)
    rank = torch.empty(n_pool, dtype=torch.int32, device=dev)
    rank[order.long()] = torch.arange(n_pool, dtype=torch.int32, device=dev)
    costs = torch.randint(0, 300, (n_pool,), generator=g, device=dev).to(torch.int16)
    idx = torch.randperm(n_pool, generator=g, device=dev)[:n]
    ws = torch.zeros(lib.dot_plan_ranked_workspace(n_pool, n, 2), dtype=torch.uint8, device=dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    wo = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    big_a = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    big_b = torch.empty_like(big_a)
    side = torch.cuda.Stream()
    t = (ctypes.c_ulonglong * 16)()
    names = "ABCDWEFG"
    for label, mode, rk, od, cst in (("positions", 0, None, None, costs), ("pool rays", 1, rank, order, costs),
                                     ("slots", 2, None, None, costs[:n].contiguous())):
        for busy in (False, True):
            for rep in range(3):
                if busy:
                    with torch.cuda.stream(side):
                        for _ in range(4):
                            big_b.copy_(big_a)
                _lib.call("dot_plan_ranked", _lib.ptr(rk), _lib.ptr(od), n_pool, _lib.ptr(idx), n, mode, _lib.ptr(cst),
                          1, _lib.ptr(wo), _lib.ptr(ws), ws.numel(), _lib.ptr(out), _lib.stream_ptr())
                torch.cuda.synchronize()
            lib.dot_diag_plan_timeline(t)
            ph = [(t[i + 1] - t[i]) / 1e3 for i in range(8)]
            print(f"{label:10s} {'beside copy' if busy else 'alone':12s} total {(t[8] - t[0]) / 1e3:7.1f} us  "
                  + " ".join(f"{names[i]} {ph[i]:6.1f}" for i in range(8)))


if __name__ == "__main__":
    main()
