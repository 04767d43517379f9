"""Summarise one ncu --set full capture into profiles/*.json (the numbers bench.py cites).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_r01_k_panel_cfg5_jt84.json \
        --launch "41st k_panel launch of one config-5 solve: jt=84, ..." --algorithmic-bytes 5505024000
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--launch", default="")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    ix = {k: i for i, k in enumerate(hdr)}
    out = {"Kernel Name": vals[ix["Kernel Name"]]}
    for k in KEYS:
        if k in ix:
            out[k] = f"{vals[ix[k]]} {units[ix[k]]}".strip()
    st = [(float(vals[i] or 0), k.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", "")) for k, i in ix.items()
          if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
    out["stalls"] = [[round(v, 3), n] for v, n in sorted(st, reverse=True)[:8]]
    if a.algorithmic_bytes:
        out["algorithmic_bytes"] = a.algorithmic_bytes
    if a.launch:
        out["launch"] = a.launch
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
