#!/usr/bin/env python
"""Attribute an ncu report's per-SASS-instruction metrics to CUDA source lines.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [--kernel comine_kernel] [--top 40]

ncu's source page gives per-instruction counters keyed by absolute SASS address; the
cubin inside libmayura.so (built with -lineinfo) gives, via `nvdisasm -g`, the source
line of every instruction offset.  The function's first address is its base.
"""
import argparse
import collections
import csv
import glob
import io
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu_sass(rep):
    if rep.endswith(".csv"):  # a `--page source --csv` export made on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kernels = []
    i = 0
    while i < len(rows):
        if rows[i] and rows[i][0] == "Kernel Name":
            name = rows[i][1]
            hdr = rows[i + 1]
            j = i + 2
            data = []
            while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
                if len(rows[j]) == len(hdr):
                    data.append(dict(zip(hdr, rows[j])))
                j += 1
            kernels.append((name, data))
            i = j
        else:
            i += 1
    return kernels


def line_map(so, mangled_hint):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True, check=True)
    cubins = glob.glob(os.path.join(tmp, "*.cubin"))
    for cb in cubins:
        dis = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
        sections = re.split(r"\n//-+ \.text\.(\S+) -+\n", dis)
        for k in range(1, len(sections), 2):
            if mangled_hint(sections[k]):
                cur = None
                mp = {}
                for ln in sections[k + 1].splitlines():
                    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                    if m:
                        cur = (os.path.basename(m.group(1)), int(m.group(2)))
                        continue
                    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
                    if m and cur:
                        mp[int(m.group(1), 16)] = cur
                return mp
    return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default="comine_kernel")
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2507_14813_b200", "lib", "libmayura.so"))
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    kernels = [(n, d) for n, d in ncu_sass(args.rep) if args.kernel in n]
    if not kernels:
        raise SystemExit("kernel not found in report")
    name, data = kernels[0]
    # mangled tag of this template instance: kernel<(int)6, (bool)1> -> kernelILi6ELb1E
    m = re.search(r"(\w+)<([^<>]*)>\(", name)
    tag = args.kernel
    if m:
        args_ = re.findall(r"\((int|bool)\)(\d+)", m.group(2))
        tag = m.group(1) + "I" + "".join(("Li%sE" if t == "int" else "Lb%sE") % v for t, v in args_)
    mp = line_map(args.so, lambda sec: tag in sec)
    base = min(int(r["Address"], 16) for r in data)
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    tot_i = tot_s = 0.0
    for r in data:
        off = int(r["Address"], 16) - base
        key = mp.get(off, ("?", 0))
        ins = float(r.get("Instructions Executed") or 0)
        smp = float(r.get("Warp Stall Sampling (All Samples)") or 0)
        agg[key][0] += ins
        agg[key][1] += smp
        tot_i += ins
        tot_s += smp
    src = {}
    for f, _ in agg:
        p = os.path.join(ROOT, "paper_2507_14813_b200", "csrc", f)
        if os.path.exists(p):
            src[f] = open(p).read().splitlines()
    print("%s\n  instructions %.3g, stall samples %.0f" % (name, tot_i, tot_s))
    print("%6s %6s  %s" % ("inst%", "stall%", "line"))
    for (f, ln), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:args.top]:
        text = src.get(f, [""] * (ln + 1))[ln - 1].strip() if ln else ""
        print("%6.2f %6.2f  %s:%d  %s" % (100 * i / tot_i, 100 * s / max(tot_s, 1), f, ln, text[:90]))


if __name__ == "__main__":
    main()
