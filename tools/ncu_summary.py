"""Summarise an ncu report (raw page) or a launch-list CSV into profiles/ (text)."""
import csv, io, re, subprocess, sys

KEYS = [r"^gpu__time_duration.sum$", r"^dram__bytes_(read|write)\.sum$", r"^dram__bytes_(read|write)\.sum\.per_second$",
        r"^gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed$", r"^launch__(grid_size|block_size|registers_per_thread|occupancy_limit_.*)$",
        r"^sm__warps_active.avg.pct_of_peak_sustained_active$", r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^l1tex__throughput.avg.pct_of_peak_sustained_elapsed$", r"^sm__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^launch__shared_mem_per_block_(dynamic|static)$", r"^smsp__inst_executed.sum$",
        r"^nvlrx__bytes.sum$", r"^nvltx__bytes.sum$",
        r"^smsp__sass_inst_executed_op_(global|shared)_(ld|st)\.sum$",
        r"^l1tex__t_(sectors|requests)_pipe_lsu_mem_global_op_(ld|st)\.sum$",
        r"^sm__ctas_launched\.sum$", r"^launch__occupancy_per_block_size$",
        r"^sm__maximum_warps_per_active_cycle_pct$", r"^launch__waves_per_multiprocessor$"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"kernel: {name}")
        for i, h in enumerate(hdr):
            if any(re.search(k, h) for k in KEYS):
                out.append(f"  {h} [{units[i]}] = {vals[i]}")
        try:
            rd = float(vals[hdr.index("dram__bytes_read.sum")]); wr = float(vals[hdr.index("dram__bytes_write.sum")])
            ur = units[hdr.index("dram__bytes_read.sum")]; uw = units[hdr.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            out.append(f"  traffic (read+write) bytes = {rd * scale[ur] + wr * scale[uw]:.0f}")
        except Exception:
            pass
    return "\n".join(out)


def launches(path):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    tot, per = 0.0, {}
    for r in rows:
        ns = float(r["Metric Value"].replace(",", ""))
        k = r["Kernel Name"].split("(")[0][:60]
        per.setdefault(k, []).append(ns)
        tot += ns
    out = [f"launches: {len(rows)}  total device time: {tot/1e3:.1f} us"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"  {k:60s} n={len(v):4d} sum={sum(v)/1e3:10.1f} us share={sum(v)/tot:6.1%} mean={sum(v)/len(v)/1e3:9.2f} us")
    return "\n".join(out)


if __name__ == "__main__":
    p = sys.argv[1]
    print(report(p) if p.endswith(".ncu-rep") else launches(p))
