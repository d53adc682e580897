"""Idle time of the GPU inside bench's timed training steps: torch.profiler
trace of 10 steps; per-stream busy intervals merged, gap = step wall - busy."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    out = os.path.join(ROOT, "gpurun_out", "trace.json")
    # --e2e: the host-fed (staged) loop instead of the resident-pool steps
    env = dict(os.environ, **({"DOT_TRACE_E2E": out} if "--e2e" in sys.argv else {"DOT_TRACE": out}))
    subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "10", "--warmup", "3",
                    "--skip-render", "--skip-refine", "--skip-cpu"], env=env, check=True,
                   stdout=subprocess.DEVNULL)
    ev = json.load(open(out))["traceEvents"]
    k = [e for e in ev if e.get("cat") == "kernel"]
    k.sort(key=lambda e: e["ts"])
    t0, t1 = k[0]["ts"], max(e["ts"] + e["dur"] for e in k)
    busy, cur_s, cur_e = 0.0, None, None
    for e in k:
        s, d = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, d
        else:
            cur_e = max(cur_e, d)
    busy += cur_e - cur_s
    print(f"kernels {len(k)}, window {t1 - t0:.0f} us, GPU busy {busy:.0f} us, idle {t1 - t0 - busy:.0f} us "
          f"({100 * (1 - busy / (t1 - t0)):.1f} %)")
    # one step's timeline (the 5th backward launch onwards)
    bw = [e for e in k if "render_bwd" in e["name"]]
    if len(bw) > 6:
        a, b = bw[5]["ts"], bw[6]["ts"]
        print("one step (us from its backward's start): stream  start  end  kernel")
        cp = [e for e in ev if e.get("cat") in ("gpu_memcpy", "gpu_memset")]
        for e in sorted(k + cp, key=lambda e: e["ts"]):
            if a - 300 <= e["ts"] < b:
                print(f"  {e.get('args', {}).get('stream', '?'):>4} {e['ts'] - a:8.0f} {e['ts'] + e['dur'] - a:8.0f}  "
                      f"{e['name'].split('(')[0][:60]}")
    # the plan's placement against the update, every step of the trace
    pl = [e for e in k if "plan_coop" in e["name"]]
    rm = [e for e in k if "rmsprop" in e["name"]]
    if pl and rm:
        rows = []
        for e in pl:
            r = min(rm, key=lambda x: abs(x["ts"] - e["ts"]))
            rows.append((e["ts"] - r["ts"], e["ts"] + e["dur"] - (r["ts"] + r["dur"]), e["dur"]))
        rows.sort()
        print("plan start - update start / plan end - update end / plan dur (us), per step:")
        print("  " + "  ".join(f"{a:.0f}/{b:.0f}/{c:.0f}" for a, b, c in rows))
    by = {}
    for e in k:
        n = e["name"].split("(")[0][:60]
        by[n] = by.get(n, 0) + e["dur"]
    for n, d in sorted(by.items(), key=lambda x: -x[1])[:8]:
        print(f"{d:9.0f} us  {n}")


if __name__ == "__main__":
    main()
