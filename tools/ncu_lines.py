"""Attribute an ncu source-page capture (SASS level) to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX CUBIN SASS_FN_REGEX [--top N] [--regions FILE]

ncu's CSV source page carries per-SASS-instruction counters (warp-level
instructions executed, stall samples by reason) but not the source line; the
line comes from `nvdisasm -g` on the same cubin (built with -lineinfo).  The
instruction offsets are matched in address order.  With --regions FILE, lines
of FILE are grouped by the nearest preceding `// ----` marker comment.
"""

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def sass_lines(cubin, fn_regex):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur = None
    pos = {}
    in_fn = False
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            in_fn = re.search(fn_regex, m.group(1)) is not None
            continue
        if not in_fn:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            pos[int(m.group(1), 16)] = cur
    return pos


def main():
    rep, kre, cubin = sys.argv[1:4]
    top = 40
    regions = None
    args = sys.argv[5:]
    if "--top" in args:
        top = int(args[args.index("--top") + 1])
    if "--regions" in args:
        regions = args[args.index("--regions") + 1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    # first line may be the kernel name
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    kname = lines[0]
    end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:end]))))  # first matching kernel only
    pos = sass_lines(cubin, sys.argv[4])
    base = int(rows[0]["Address"], 16)
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    agg = defaultdict(lambda: defaultdict(float))
    tot = defaultdict(float)
    nomap = 0
    for r in rows:
        off = int(r["Address"], 16) - base
        key = pos.get(off)
        if key is None:
            nomap += 1
            key = ("?", 0)
        a = agg[key]
        a["inst"] += float(r["Instructions Executed"] or 0)
        a["wf"] += float(r.get("L1 Wavefronts Shared") or 0)
        a["wfi"] += float(r.get("L1 Wavefronts Shared Ideal") or 0)
        tot["wf"] += float(r.get("L1 Wavefronts Shared") or 0)
        a["samples"] += float(r["Warp Stall Sampling (All Samples)"] or 0)
        for c in stall_cols:
            a[c] += float(r[c] or 0)
        tot["inst"] += float(r["Instructions Executed"] or 0)
        tot["samples"] += float(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"kernel: {kname[:160]}")
    print(f"sass rows {len(rows)}, unmapped {nomap}; total inst {tot['inst']:.4g}, samples {tot['samples']:.4g}, "
          f"shared wavefronts {tot['wf']:.4g}")
    src_cache = {}

    def src(f, l):
        if f not in src_cache:
            try:
                src_cache[f] = open(f).read().splitlines()
            except OSError:
                src_cache[f] = []
        s = src_cache[f]
        return s[l - 1].strip()[:70] if 0 < l <= len(s) else ""

    if regions:
        text = open(regions).read().splitlines()
        marker = {}
        cur = "head"
        for i, t in enumerate(text, 1):
            mm = re.search(r"// ----\s*(.*)", t)
            if mm:
                cur = mm.group(1)[:60]
            marker[i] = cur
        ragg = defaultdict(lambda: defaultdict(float))
        for (f, l), a in agg.items():
            name = marker.get(l, "?") if f.endswith(regions.split("/")[-1]) else "other:" + f.split("/")[-1]
            for k, v in a.items():
                ragg[name][k] += v
        print(f"\n{'region':62s} {'inst%':>6s} {'samp%':>6s} {'smem wf%':>8s} {'(ideal)':>8s}  top stalls")
        for name, a in sorted(ragg.items(), key=lambda kv: -kv[1]["samples"]):
            st = sorted(((a[c], c[6:]) for c in stall_cols), reverse=True)[:4]
            sts = " ".join(f"{n}:{100 * v / max(a['samples'], 1):.0f}" for v, n in st if v > 0)
            print(f"{name:62s} {100 * a['inst'] / tot['inst']:6.1f} {100 * a['samples'] / tot['samples']:6.1f} "
                  f"{100 * a['wf'] / max(tot['wf'], 1):8.1f} {100 * a['wfi'] / max(tot['wf'], 1):8.1f}  {sts}")
    key = "wf" if "--by-wf" in args else "samples"
    print(f"\n{'file:line':28s} {'inst%':>6s} {'samp%':>6s} {'wf%':>6s}  top stalls | source")
    for (f, l), a in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        st = sorted(((a[c], c[6:]) for c in stall_cols), reverse=True)[:3]
        sts = " ".join(f"{n}:{100 * v / max(a['samples'], 1):.0f}" for v, n in st if v > 0)
        print(f"{f.split('/')[-1] + ':' + str(l):28s} {100 * a['inst'] / tot['inst']:6.1f} "
              f"{100 * a['samples'] / tot['samples']:6.1f} {100 * a['wf'] / max(tot['wf'], 1):6.1f}  {sts:32s} | {src(f, l)}")


if __name__ == "__main__":
    main()
