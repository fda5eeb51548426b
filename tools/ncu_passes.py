"""Per-pass R2 roofline of the staged 2D passes from an ncu metrics CSV of
one forward + backward of a 2D config (tools/profile_round.sh: `ncu --metrics ... --csv
python tools/profile_step.py c5 1`).

    python tools/ncu_passes.py <csv> <tag> [C5]

For every pass: ncu DRAM bytes and duration -> GB/s and the fraction of the measured HBM
peak, next to the pass's REQUIRED staged bytes (12.25 B/px cold row/column pass, 16.5 B/px
warm passes, 12.5 B/px the last column pass; adjoint passes 8.25 B/px for the first two,
12.25 B/px after).  Writes profiles/ncu_passes_c5.json (read by
bench.py as r2_per_pass_c5) and profiles/<tag>_passes_c5.md.
"""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
      "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    path, tag = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    hdr = rows[hi]
    ii, ki, mi, ui, vi = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"kernel": r[ki]})
        try:
            d[r[mi]] = float(r[vi].replace(",", "")) * SC.get(r[ui], 1.0)
        except ValueError:
            pass
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    cfg = sys.argv[3] if len(sys.argv) > 3 else "C5"
    N, C, H, W, K = {"C5": (256, 3, 224, 224, 4), "C4": (16, 3, 512, 512, 4), "C3": (64, 64, 56, 56, 4)}[cfg]
    px = N * C * H * W
    fwd = [d for d in launches.values() if any(k in d["kernel"] for k in ("k_row_fwd<", "k_row_fwd_r<", "k_col_fwd<"))]
    bwd = [d for d in launches.values() if any(k in d["kernel"] for k in ("k_row_bwd<", "k_row_bwd_r<", "k_row_bwd_w<", "k_col_bwd<"))]
    out = []
    for j, d in enumerate(fwd[:2 * K]):
        k, col = j // 2 + 1, j % 2 == 1
        req = 12.25 if k == 1 else (12.5 if (col and k == K) else 16.5)
        out.append(("fwd", ("col" if col else "row") + str(k), d, req))
    for j, d in enumerate(bwd[:2 * K]):
        k, col = K - j // 2, j % 2 == 0
        req = 8.25 if j < 2 else 12.25
        out.append(("bwd", ("col" if col else "row") + str(k), d, req))
    table, js = [], []
    for direction, name, d, req in out:
        byt = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        t = d.get("gpu__time_duration.sum", 0)
        gbs = byt / t / 1e9 if t else 0
        e = {"dir": direction, "pass": name, "kernel": d["kernel"][:60], "us": t * 1e6, "dram_bytes": byt,
             "dram_GBps": gbs, "frac_of_peak": gbs / peak, "required_bytes": req * px,
             "required_frac_of_peak": (req * px / t / 1e9 / peak) if t else None,
             "warp_instr": d.get("smsp__inst_executed.sum"),
             "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active")}
        js.append(e)
        table.append("| %s | %s | %.1f | %.1f | %.0f | %.3f | %.2f | %.3f | %.3g | %.1f |" % (
            direction, name, e["us"], byt / 1e6, gbs, e["frac_of_peak"], req, e["required_frac_of_peak"] or 0,
            e["warp_instr"] or 0, e["issue_active_pct"] or 0))
    doc = {"config": "%s %dx%dx%dx%d fp32, K=%d, staged passes (default path)" % (cfg, N, C, H, W, K),
           "peak_GBps": peak,
           "source": "profiles/%s_passes_%s.md (ncu --metrics, --clock-control none, one fwd + one bwd)" % (tag, cfg.lower()),
           "passes": js}
    with open(os.path.join(ROOT, "profiles", "ncu_passes_%s.json" % cfg.lower()), "w") as f:
        json.dump(doc, f, indent=1)
    md = ["# Per-pass R2 roofline, %s (%s)" % (cfg, tag), "",
          "ncu `gpu__time_duration`, `dram__bytes_read/write`, `smsp__inst_executed`, issue active, one launch per "
          "pass (cold L2, serialised).  Peak %.0f GB/s (MEASURED_PEAKS.json).  `req B/px`: the bytes the pass "
          "must move when staged (DESIGN.md section 7); `req frac` = those bytes over the pass time." % peak, "",
          "| dir | pass | us | DRAM MB | GB/s | frac | req B/px | req frac | warp instr | issue % |",
          "|---|---|---|---|---|---|---|---|---|---|"] + table
    with open(os.path.join(ROOT, "profiles", "%s_passes_%s.md" % (tag, cfg.lower())), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
