"""Turn a tools/capture_profiles.sh run into committed evidence under profiles/.

    python tools/summarise_profiles.py <tag>

Writes profiles/<tag>_bench.json (the bench line), profiles/<tag>_launch_shares.txt
(per-kernel share of the timed steps from the ncu launch list),
profiles/<tag>_ncu_full.txt (key --set full metrics + stall breakdown per
kernel) and updates profiles/traffic.json (DRAM bytes per launch of the
dominant kernels, read by bench.py for roofline.traffic)."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
        "smsp__inst_executed_op_global_red.sum", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sass__inst_executed_register_spilling", "lts__t_sectors.sum",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum"]


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) > vi:
            k = r[ki].split("(")[0]
            k = k.replace("void ", "")[:80]
            agg[k] += float(r[vi].replace(",", ""))
            cnt[k] += 1
    tot = sum(agg.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off "
             f"(timed steps only; cold-cache serialised launches: compare shares)",
             f"# total {tot / 1e3:.1f} us over the captured steps"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"{v / 1e3:10.1f} us {cnt[k]:4d}x {100 * v / tot:5.1f}%  {k}")
    return "\n".join(lines) + "\n", agg, cnt


def full_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        m = {}
        for k in KEYS:
            if k in h:
                m[k] = (r[h.index(k)], units[h.index(k)])
        stalls = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                except ValueError:
                    pass
        out.append((name, m, stalls))
    return out


def refine_totals(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    mi, vi, ui, idi = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    t = b = 0.0
    ids = set()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        ids.add(r[idi])
        if r[mi] == "gpu__time_duration.sum":
            t += v * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(r[ui], 1.0)
        elif r[mi].startswith("dram__bytes_"):
            b += to_bytes(r[vi], r[ui])
    return t, b, len(ids)


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    tag = sys.argv[1]
    src = os.path.join(ROOT, "gpurun_out", f"prof_{tag}")
    prof = os.path.join(ROOT, "profiles")
    bench = open(os.path.join(src, "bench.json")).read().strip().splitlines()[-1]
    json.loads(bench)
    open(os.path.join(prof, f"{tag}_bench.json"), "w").write(bench + "\n")
    text, agg, cnt = launch_shares(os.path.join(src, "launches.csv"))
    open(os.path.join(prof, f"{tag}_launch_shares.txt"), "w").write(text)
    full = full_metrics(os.path.join(src, "full.ncu-rep"))
    if os.path.exists(os.path.join(src, "render_full.ncu-rep")):
        full += full_metrics(os.path.join(src, "render_full.ncu-rep"))
    lines = [f"# ncu --set full --clock-control none, first timed launch of each kernel ({tag})"]
    traffic_path = os.path.join(prof, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for name, m, stalls in full:
        short = name.split("(")[0].replace("void ", "")
        lines.append(f"\n## {short}")
        for k, (v, u) in m.items():
            lines.append(f"  {k:70s} {v} {u}")
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda x: -x[1])[:8]
        lines.append("  stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))
        rd = to_bytes(*m["dram__bytes_read.sum"])
        wr = to_bytes(*m["dram__bytes_write.sum"])
        key = "render_bwd_buffered" if "render_bwd_buffered" in short else short.split("<")[0].split("::")[-1]
        if "lts__t_sector_hit_rate.pct" in m:
            traffic_hit = float(m["lts__t_sector_hit_rate.pct"][0])
        else:
            traffic_hit = None
        def pct(k):
            return float(m[k][0].replace(",", "")) if k in m else None

        traffic[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                        "l2_hit_pct": traffic_hit, "capture": f"profiles/{tag}_ncu_full.txt", "kernel": short,
                        "ncu_time_s": float(m["gpu__time_duration.sum"][0].replace(",", "")) *
                        {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
                         "nsecond": 1e-9}.get(m["gpu__time_duration.sum"][1], 1.0),
                        "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                        "fp64_pipe_pct": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                        "xu_pipe_pct": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                        "lsu_pipe_pct": pct("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                        "warps_active_pct": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
                        "l2_bytes_per_launch": 32.0 * float(m["lts__t_sectors.sum"][0].replace(",", ""))
                        if "lts__t_sectors.sum" in m else None}
    refine_csv = os.path.join(src, "refine_launches.csv")
    if os.path.exists(refine_csv):  # one refine pass: every launch's time and DRAM bytes
        res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "refine_launches.py"), refine_csv],
                             capture_output=True, text=True)
        open(os.path.join(prof, f"{tag}_refine_launches.txt"), "w").write(res.stdout)
        tot_t, tot_b, n = refine_totals(refine_csv)
        traffic["refine_pass"] = {"dram_bytes_per_launch": tot_b, "ncu_time_s": tot_t, "launches": n,
                                  "capture": f"profiles/{tag}_refine_launches.txt",
                                  "kernel": "one configs[4] refine pass (all launches)"}
        lines.append("\n## refine pass (configs[4])\n" + res.stdout)
    open(os.path.join(prof, f"{tag}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print(text)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
