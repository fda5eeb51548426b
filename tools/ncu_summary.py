"""Summarise ncu captures (raw CSV pages) and a launch list into profiles/.

    python tools/ncu_summary.py <gpurun_out dir> <round tag>

Writes profiles/<tag>_ncu_summary.md, profiles/<tag>_launches.md and
profiles/ncu_traffic.json (per-launch DRAM bytes bench.py reports as `traffic`).
"""
import csv
import glob
import json
import os
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instr executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "LDS executed"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % peak"),
]
STALLS = ["no_instruction", "wait", "long_scoreboard", "short_scoreboard", "branch_resolving",
          "math_pipe_throttle", "barrier", "mio_throttle", "lg_throttle", "not_selected", "dispatch_stall"]


def read_raw(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def fnum(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def summarize(d, name):
    out = {"name": name}
    for k, label in KEYS:
        if k in d:
            out[label] = (fnum(d[k][0]), d[k][1])
    st = {}
    for s in STALLS:
        k = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s
        if k in d:
            st[s] = fnum(d[k][0])
    out["stalls"] = st
    out["kernel"] = d.get("Kernel Name", ("?", ""))[0]
    return out


def main():
    src, tag = sys.argv[1], sys.argv[2]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prof = os.path.join(root, "profiles")
    os.makedirs(prof, exist_ok=True)
    lines = ["# ncu --set full summaries (%s)" % tag, "",
             "One capture per kernel (`tools/ncu_capture.sh`, `--clock-control none`, cold L2, serialised).",
             "Durations are ncu's; bench.py's live CUDA-event timings are the reported numbers.", ""]
    traffic = {}
    pipe_info = {}
    warp_instr = {}
    for raw in sorted(glob.glob(os.path.join(src, "%s_*.raw.csv" % tag))):
        name = os.path.basename(raw).replace(".raw.csv", "")
        d = read_raw(raw)
        if not d:
            continue
        s = summarize(d, name)
        if "warp instr executed" in s and s["warp instr executed"][0]:
            warp_instr[name] = s["warp instr executed"][0]
        pipe_info[name] = {lab: s[lab][0] for lab in ("issue active %", "ALU pipe % peak", "FMA pipe % peak",
                                                        "achieved occupancy %") if lab in s}
        lines.append("## %s" % name)
        lines.append("")
        lines.append("`%s`" % s["kernel"][:160])
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for _, label in KEYS:
            if label in s:
                v, u = s[label]
                lines.append("| %s | %s | %s |" % (label, "%.4g" % v if v is not None else "-", u))
        if "dram read" in s and "dram write" in s:
            tot = (s["dram read"][0] or 0) * (1 if s["dram read"][1] == "byte" else 1)
            unit_r = s["dram read"][1]
            unit_w = s["dram write"][1]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tb = (s["dram read"][0] or 0) * scale.get(unit_r, 1) + (s["dram write"][0] or 0) * scale.get(unit_w, 1)
            dur = s.get("duration", (None, ""))
            dscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
                      "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
            secs = (dur[0] or 0) * dscale.get(dur[1], 1e-9)
            lines.append("| DRAM bytes (read+write) | %.4g | byte |" % tb)
            if secs:
                lines.append("| DRAM GB/s (ncu) | %.1f | GB/s |" % (tb / secs / 1e9))
            traffic[name] = tb
        lines.append("")
        lines.append("stall reasons (warps per issue): " + ", ".join(
            "%s %.2f" % (k, v) for k, v in sorted(s["stalls"].items(), key=lambda kv: -(kv[1] or 0)) if v and v > 0.02))
        lines.append("")
    with open(os.path.join(prof, "%s_ncu_summary.md" % tag), "w") as f:
        f.write("\n".join(lines) + "\n")
    tjp = os.path.join(prof, "ncu_traffic.json")
    try:
        with open(tjp) as f:
            tj = json.load(f)            # merge: a capture set without C2 keeps the C2 keys
    except Exception:
        tj = {}
    for name, pipes in pipe_info.items():
        if name.endswith("c2_row_fwd"):
            tj["c2_fwd_pipes"] = pipes
        elif name.endswith("c2_row_bwd"):
            tj["c2_bwd_pipes"] = pipes
    # executed warp instructions per launch of the C2 forward op (coarse pre-pass + fine PN)
    wi = {n: v for n, v in warp_instr.items() if n.endswith(("c2_row_fwd", "c2_coarse"))}
    if wi:
        tj["c2_fwd_warp_instr_per_launch"] = sum(wi.values())
    byk = {}
    for k, v in traffic.items():
        if k.endswith("c2_row_fwd"):
            tj["c2_fwd_bytes_per_launch"] = v
            byk["k_row_fwd_w (fine projected Newton)"] = v
        elif k.endswith("c2_coarse"):
            byk["k_coarse_rows4 (coarse pre-pass)"] = v
        elif k.endswith("c2_row_bwd"):
            tj["c2_bwd_bytes_per_launch"] = v
        else:
            tj[k] = v
    if byk:
        # DRAM bytes of EVERY kernel of the C2 forward op (roofline.traffic in bench.py)
        tj["c2_fwd_bytes_by_kernel"] = byk
        tj["c2_fwd_op_bytes_per_launch"] = sum(byk.values())
        tj["source"] = "profiles/%s_ncu_summary.md (ncu --set full, one launch each)" % tag
    with open(tjp, "w") as f:
        json.dump(tj, f, indent=1)
    # launch list
    ll = glob.glob(os.path.join(src, "launches_%s.csv" % tag))
    if ll:
        rows = list(csv.reader(open(ll[0])))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hi]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = defaultdict(list)
        for r in rows[hi + 1:]:
            v = fnum(r[vi])
            if v is not None:
                agg[r[ki]].append(v)
        tot = sum(sum(v) for v in agg.values())
        out = ["# Launch list (%s): `ncu --metrics gpu__time_duration.sum --clock-control none` of "
               "`python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-verify`" % tag, "",
               "Serialised, cold-cache per-launch times: compare SHARES, not absolutes.", "",
               "| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            out.append("| `%s` | %d | %.3f | %.1f | %.1f%% |" % (k[:90], len(v), sum(v) / 1e6, sum(v) / len(v) / 1e3,
                                                              100 * sum(v) / tot))
        with open(os.path.join(prof, "%s_launches.md" % tag), "w") as f:
            f.write("\n".join(out) + "\n")
    print("wrote profiles/%s_*" % tag)


if __name__ == "__main__":
    main()
