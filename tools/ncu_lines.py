"""Attribute an ncu --set full capture's per-instruction samples to CUDA source lines.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep k_panel 'k_panelILb1ELb1ELb1E' [--top 40]

Maps the SASS addresses of the captured kernel (ncu --page source) to file:line
through nvdisasm -g line info of the in-tree libhsrq_b200.so (which must be the
binary that was profiled) and prints the hottest lines by stall samples.
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2101_05063_b200", "libhsrq_b200.so")


def sass_lines(func_pat, outer=False):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, check=True, capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cubin)], check=True,
                         capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(out) if l.startswith(".text.") and re.search(func_pat, l)]
    if not start:
        raise SystemExit(f"no function matching {func_pat}")
    i0 = start[0]
    i1 = next((i for i in range(i0 + 1, len(out)) if out[i].startswith(".text.")), len(out))
    cur, m2l = None, {}
    for l in out[i0:i1]:
        if l.strip().startswith("//## File"):
            locs = re.findall(r'"([^"]+)", line (\d+)', l)
            f, ln = locs[-1] if outer else locs[0]
            cur = (os.path.basename(f), int(ln))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            m2l[int(m.group(1), 16)] = cur
    return m2l


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel", help="regex of the kernel name as ncu shows it")
    ap.add_argument("func", help="regex of the mangled SASS function name")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--outer", action="store_true",
                    help="attribute inlined code to its outermost call site")
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{a.kernel}"], check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = [i for i, r in enumerate(rows) if len(r) > 3 and r[0] == "Address"][0]
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    m2l = sass_lines(a.func, a.outer)
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    base = None
    ti = ts = 0.0
    for r in rows[hi + 1:]:
        if len(r) < len(h) or not r[0].startswith("0x"):
            continue
        ad = int(r[0], 16)
        base = ad if base is None else base
        ie = float(r[ix["Instructions Executed"]] or 0)
        sm = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        k = m2l.get(ad - base, ("?", 0))
        agg[k][0] += ie
        agg[k][1] += sm
        ti += ie
        ts += sm
    srcs = {}
    for d in ("paper_2101_05063_b200/csrc",):
        for f in os.listdir(os.path.join(ROOT, d)):
            srcs[f] = open(os.path.join(ROOT, d, f)).read().split("\n")
    print(f"instructions {ti:.0f}, stall samples {ts:.0f}")
    for (f, ln), (ie, sm) in sorted(agg.items(), key=lambda x: -x[1][1])[: a.top]:
        text = srcs[f][ln - 1].strip()[:90] if f in srcs and 0 < ln <= len(srcs[f]) else ""
        print(f"{100 * sm / ts:5.1f}% samples {100 * ie / ti:5.1f}% inst  {f}:{ln}  {text}")


if __name__ == "__main__":
    main()
