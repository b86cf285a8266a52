"""Top source lines by warp-stall samples from an ncu report
(ncu --page source --print-source cuda,sass CSV).

  python tools/ncu_src.py report.ncu-rep kernel_regex|#launch_index [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
# kern "#K" selects the report's K-th profiled launch instead of a name regex
sel = (["--launch-skip", kern[1:], "--launch-count", "1"] if kern.startswith("#")
       else ["--kernel-name", "regex:" + kern])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + sel,
                     capture_output=True, text=True).stdout
fname, hdr, data = None, None, []
stall_cols = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if hdr is None or not r[0] or len(r) < 8:
        continue
    try:
        w = float(r[4] or 0)
    except ValueError:
        continue
    stalls = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols if r[i] not in ("", "-")), reverse=True)[:3]
    data.append((w, fname, r[0], r[1].strip()[:90], r[7], stalls))
tot = sum(d[0] for d in data) or 1
data.sort(key=lambda d: -d[0])
print(f"total samples {tot:.0f}")
for w, f, ln, src, inst, st in data[:top]:
    s = " ".join(f"{n}:{100 * v / w:.0f}%" for v, n in st if w)
    print(f"{100 * w / tot:5.1f}% {f}:{ln:<5} inst={inst:>11} [{s}] {src}")
