"""Host time of the cooperative plan launch (dot_plan_ranked) when the GPU
is idle vs busy with a long grid on another stream (a full-GPU elementwise
kernel) -- does cudaLaunchCooperativeKernel block the host?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2307_15333_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    dev = torch.device("cuda")
    n_pool, n = 1 << 26, 1 << 20
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    idx = torch.randperm(n_pool, generator=g, device=dev)[:n]
    costs = torch.randint(0, 300, (n_pool,), generator=g, device=dev).to(torch.int16)
    ws = torch.zeros(lib.dot_plan_ranked_workspace(n_pool, n, 0), dtype=torch.uint8, device=dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    wo = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    big = torch.empty(1 << 29, dtype=torch.float32, device=dev)
    side = torch.cuda.Stream()

    def launch(stream):
        _lib.call("dot_plan_ranked", None, None, n_pool, _lib.ptr(idx), n, 0, _lib.ptr(costs), 1, _lib.ptr(wo),
                  _lib.ptr(ws), ws.numel(), _lib.ptr(out), _lib.stream_ptr(stream))

    for label, busy, same in (("idle", False, False), ("busy other stream", True, False),
                              ("busy same stream", True, True)):
        ts = []
        for rep in range(10):
            torch.cuda.synchronize()
            if busy:
                with torch.cuda.stream(side if not same else torch.cuda.current_stream()):
                    for _ in range(20):
                        big.mul_(1.0000001)
            t0 = time.perf_counter()
            launch(torch.cuda.current_stream())
            ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        ts.sort()
        print(f"{label:20s} host launch median {1e6 * ts[5]:8.1f} us  max {1e6 * ts[-1]:8.1f} us")


if __name__ == "__main__":
    main()
