"""Per-kernel summary of ncu --set full reports -> JSON (profiles/<round>/
ncu_summary.json; bench.py reads dram bytes per launch from it).

  python tools/ncu_summary.py OUT.json LABEL=report.ncu-rep[:kernel_regex] ...

Each entry is keyed "<kernel template>:<LABEL>" and records the launch's
duration, DRAM bytes read / written, L2 hit rate, warps active, issue
activity, instructions, registers and grid, plus the git SHA of the build."""
import csv
import io
import json
import re
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
FIELDS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warp_instructions": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}


def short(name: str) -> str:
    m = re.search(r"(\w+)(<[^>]*>)?\(", name)
    base = m.group(1) if m else name
    tmpl = re.sub(r"\s+", "", m.group(2)) if m and m.group(2) else ""
    tmpl = re.sub(r"\(\w+\)", "", tmpl)
    return base + tmpl


def main():
    out = sys.argv[1]
    try:
        with open(out) as f:
            doc = json.load(f)
    except Exception:
        doc = {"kernels": {}}
    import os
    sha = os.environ.get("GIT_SHA") or subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True,
                                                      text=True).stdout.strip()
    for arg in sys.argv[2:]:
        label, spec = arg.split("=", 1)
        rep, _, kre = spec.partition(":")
        text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(text)))
        hdr, units = rows[0], rows[1]
        idx = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            name = r[idx["Kernel Name"]]
            if kre and not re.search(kre, name):
                continue
            e = {"git": sha, "report": rep}
            for k, metric in FIELDS.items():
                if metric not in idx:
                    continue
                v = r[idx[metric]].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                e[k] = x * SCALE.get(units[idx[metric]], 1.0) if k in ("duration_ms", "dram_bytes_read",
                                                                          "dram_bytes_write") else x
            doc["kernels"][f"{short(name)}:{label}"] = e
    with open(out, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
    print(json.dumps(doc, indent=1)[:3000])


if __name__ == "__main__":
    main()
