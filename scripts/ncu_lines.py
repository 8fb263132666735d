"""Per-source-line warp-stall samples of an ncu --set full report (--import-source on).

python scripts/ncu_lines.py report.ncu-rep [top]   (run here; no GPU needed)
Prints the lines with the most samples and their dominant stall reasons.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[2:], rec[2:]))
    d["_file"], d["_line"], d["_src"] = fname, rec[0], rec[1]
    rows.append(d)
def num(v):
    try:
        return int(float(v))
    except (TypeError, ValueError):
        return 0


stalls = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
total = sum(num(r.get("Warp Stall Sampling (All Samples)")) for r in rows)
rows.sort(key=lambda r: -num(r.get("Warp Stall Sampling (All Samples)")))
print("total samples", total)
for r in rows[:top]:
    s = num(r.get("Warp Stall Sampling (All Samples)"))
    st = sorted(((num(r.get(h)), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{s:7d} {100.0 * s / max(total, 1):5.1f}% {r['_file']}:{r['_line']:>5} "
          + " ".join(f"{n}={v}" for v, n in st if v) + "  | " + r["_src"].strip()[:70])
