"""Summarise gpurun_out ncu artefacts into a markdown file under profiles/.

    python tools/ncu_summary.py OUT.md [launches.csv] [rep.ncu-rep ...]
"""
import collections
import csv
import gzip
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    opener = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(opener(path, "rt")))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ni = hdr.index("Metric Name")
    tot, cnt, dram = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("dpn::(anonymous namespace)::", "")
        v = float(r[mi].replace(",", ""))
        if r[ni].startswith("dram__bytes"):
            dram[name] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1.0)
            continue
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    out = [f"launch list `{path}`: {sum(cnt.values())} launches, {s / 1e3:.1f} ms serialised "
           "(ncu, cold cache: compare shares, not absolutes)", "",
           "| kernel | launches | total ms | share | DRAM GB (r+w) | DRAM GB/s while running |",
           "|---|---|---|---|---|---|"]
    for k, v in tot.most_common(20):
        gb = dram[k] / 1e9
        out.append(f"| `{k[:70]}` | {cnt[k]} | {v / 1e3:.2f} | {100 * v / s:.1f}% | "
                   f"{gb:.1f} | {gb / (v / 1e6) if v else 0:.0f} |")
    return out


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return [f"`{path}`: no kernels captured", ""]
    hdr, units = rows[0], rows[1]
    if any(m not in hdr for m in METRICS):
        return [f"`{path}`: metrics missing ({[m for m in METRICS if m not in hdr]})", ""]
    idx = [hdr.index(m) for m in METRICS]
    ki = hdr.index("Kernel Name")
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0,
             "msecond": 1e3}

    def val(r, i):
        return float(r[i] or 0) * scale.get(units[i], 1.0)
    out = [f"`{path}` (ncu --set full):", "",
           "| kernel | us | tensor % | DRAM rd MB | DRAM wr MB | DRAM % | grid | regs | warps % |",
           "|---|---|---|---|---|---|---|---|---|"]
    for r in rows[2:]:
        v = [r[i] for i in idx]
        out.append(f"| `{r[ki].split('(')[0][-60:]}` | {val(r, idx[0]):.1f} | {float(v[1] or 0):.1f} | "
                   f"{val(r, idx[2]):.1f} | {val(r, idx[3]):.1f} | {float(v[4]):.1f} | {v[5]} | {v[6]} | "
                   f"{float(v[7]):.1f} |")
    return out


def main():
    out_md, paths = sys.argv[1], sys.argv[2:]
    lines = []
    for p in paths:
        lines += (launches(p) if p.endswith((".csv", ".csv.gz")) else report(p)) + [""]
    open(out_md, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
