"""Summarise ncu captures into committed evidence (run in the build container).

    python profiles/summarize.py <report.ncu-rep> <workload> <out.txt>
        -> writes the key metrics + top stall reasons + hottest SASS lines of the
           k_spmv launch, and records dram read+write bytes per launch in
           profiles/ncu_traffic.json (read by bench.py for roofline.traffic)
    python profiles/summarize.py --launches <launches.csv> <out.txt>
        -> per-kernel share of device time from the `--metrics
           gpu__time_duration.sum` launch list
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__shared_mem_config_size", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
    "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def summarize(rep, workload, out_txt):
    rows = ncu_csv(rep, "raw")
    hdr, units = rows[0], rows[1]
    lines = [f"ncu --set full summary: {os.path.basename(rep)} (workload {workload})"]
    kname = hdr.index("Kernel Name")
    for d in rows[2:]:
        if "k_spmv" not in d[kname]:
            continue
        lines.append(f"kernel: {d[kname]}")
        for k in KEYS:
            if k in hdr:
                lines.append(f"  {k:58s} {d[hdr.index(k)]:>16s} {units[hdr.index(k)]}")
        rd = to_bytes(d[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(d[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        lines.append(f"  dram read+write per launch: {rd + wr:.0f} bytes")
        stalls = sorted(((float(d[i]), h) for i, h in enumerate(hdr)
                         if h.startswith("smsp__pcsamp_warps_issue_stalled") and
                         not h.endswith("not_issued") and d[i].replace(".", "").isdigit()),
                        reverse=True)[:8]
        lines.append("  top warp-stall samples:")
        lines += [f"    {v:10.0f} {h}" for v, h in stalls]
        path = os.path.join(HERE, "ncu_traffic.json")
        t = json.load(open(path)) if os.path.exists(path) else {}
        t[workload] = {"k_spmv_dram_bytes": rd + wr, "report": os.path.basename(rep)}
        json.dump(t, open(path, "w"), indent=1, sort_keys=True)
        break
    src = ncu_csv(rep, "source")
    h2 = src[1]
    iss = h2.index("Warp Stall Sampling (All Samples)")
    isrc = h2.index("Source")
    iex = h2.index("Instructions Executed")
    body = [r for r in src[2:] if len(r) > iss and r[iss].isdigit()]
    tot = sum(int(r[iss]) for r in body) or 1
    lines.append(f"  hottest SASS (stall samples, share of {tot}):")
    for r in sorted(body, key=lambda r: -int(r[iss]))[:12]:
        lines.append(f"    {int(r[iss]):7d} {100 * int(r[iss]) / tot:5.1f}%  exec={r[iex]:>9s}  {r[isrc].strip()[:70]}")
    with open(out_txt, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


CONV_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
             "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
             "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
             "launch__block_size", "launch__registers_per_thread"]


def kernels(rep, workload, out_txt):
    """Every captured launch (converter kernels): duration, DRAM bytes and
    achieved DRAM GB/s, L2 hit rate, top stall."""
    rows = ncu_csv(rep, "raw")
    hdr, units = rows[0], rows[1]
    kname = hdr.index("Kernel Name")
    lines = [f"ncu --set full, converter kernels: {os.path.basename(rep)} (workload {workload})"]
    for d in rows[2:]:
        name = d[kname].split("(")[0].replace("void ", "")
        lines.append(f"kernel: {name}")
        for k in CONV_KEYS:
            if k in hdr:
                lines.append(f"  {k:58s} {d[hdr.index(k)]:>16s} {units[hdr.index(k)]}")
        rd = to_bytes(d[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(d[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        t = float(d[hdr.index("gpu__time_duration.sum")]) * {
            "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(units[hdr.index("gpu__time_duration.sum")], 1e-9)
        lines.append(f"  dram read+write {rd + wr:.0f} bytes -> {(rd + wr) / t / 1e9:.0f} GB/s")
        stalls = sorted(((float(d[i]), h) for i, h in enumerate(hdr)
                         if h.startswith("smsp__pcsamp_warps_issue_stalled") and
                         not h.endswith("not_issued") and d[i].replace(".", "").isdigit()),
                        reverse=True)[:3]
        lines.append("  top stalls: " + ", ".join(f"{h.split('stalled_')[1]}={v:.0f}" for v, h in stalls))
    with open(out_txt, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(csv_path, out_txt):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = {}
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
        c, s = per.get(name, (0, 0.0))
        per[name] = (c + 1, s + v)
    tot = sum(s for _, s in per.values())
    lines = [f"ncu launch list ({os.path.basename(csv_path)}): kernel, launches, total us, share"]
    for name, (c, s) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"  {name[:70]:70s} {c:5d} {s:12.1f} {100 * s / tot:6.2f}%")
    with open(out_txt, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "--kernels":
        kernels(sys.argv[2], sys.argv[3], sys.argv[4])
    elif sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarize(sys.argv[1], sys.argv[2], sys.argv[3])
