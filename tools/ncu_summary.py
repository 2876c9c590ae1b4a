"""Summarise `ncu --set full` reports (one kernel launch each) into a markdown
table: duration, DRAM traffic and bandwidth, SM / tensor / memory throughput,
occupancy, registers, top warp-stall reasons.  Usage: ncu_summary.py rep..."""
import csv
import io
import subprocess
import sys

KEYS = {
    "dur_us": ("gpu__time_duration.sum", 1e-3),
    "dram_rd_MB": ("dram__bytes_read.sum", None),
    "dram_wr_MB": ("dram__bytes_write.sum", None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "regs": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
}


def raw_all(rep):
    """One dict per profiled launch in the report."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, vals)} for vals in rows[2:] if len(vals) == len(hdr)]


def raw(rep):
    return raw_all(rep)[0]


def stalls_raw(d, top=3):
    pre = "smsp__pcsamp_warps_issue_stalled_"
    agg = {}
    for k, (v, _) in d.items():
        if k.startswith(pre) and not k.endswith("_not_issued"):
            try:
                agg[k[len(pre):]] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(agg.values()) or 1.0
    best = sorted(agg.items(), key=lambda kv: -kv[1])[:top]
    return ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in best)


def num(d, key):
    v, u = d.get(key, ("nan", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return float("nan"), u
    return x, u


def to_mb(x, u):
    return x * {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}.get(u, 1e-6)


def to_us(x, u):
    return x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1e-3)


def stalls(rep, top=3):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return ""
    hdr = rows[1]
    st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = {}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        for i in st:
            try:
                agg[hdr[i]] = agg.get(hdr[i], 0.0) + float(r[i])
            except ValueError:
                pass
    tot = sum(agg.values()) or 1.0
    best = sorted(agg.items(), key=lambda kv: -kv[1])[:top]
    return ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in best)


def main(reps):
    print("| kernel | µs | DRAM rd MB | DRAM wr MB | DRAM GB/s | DRAM % | SM % | tensor % | L2 % | warps % | regs | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for rep in reps:
      launches = raw_all(rep)
      for d in launches:
        name = rep.split("/")[-1].replace(".ncu-rep", "")
        if len(launches) > 1:
            kn = d.get("Kernel Name", ("?", ""))[0]
            name = kn.replace("void ", "").replace("<unnamed>::", "").split("(")[0]
        us = to_us(*num(d, "gpu__time_duration.sum"))
        rd = to_mb(*num(d, "dram__bytes_read.sum"))
        wr = to_mb(*num(d, "dram__bytes_write.sum"))
        gbs = (rd + wr) * 1e-3 / (us * 1e-6) if us > 0 else float("nan")
        f = lambda k: num(d, KEYS[k][0])[0]   # noqa: E731
        print(f"| {name} | {us:.1f} | {rd:.1f} | {wr:.1f} | {gbs:.0f} | {f('dram_pct'):.1f} | {f('sm_pct'):.1f} | "
              f"{f('tensor_pct'):.1f} | {f('l2_pct'):.1f} | {f('warps_pct'):.1f} | {f('regs'):.0f} | "
              f"{stalls(rep) if len(launches) == 1 else stalls_raw(d)} |")


if __name__ == "__main__":
    main(sys.argv[1:])
