"""Per-launch DRAM bytes / duration of one kernel from an ncu --set full report -> JSON.

python scripts/ncu_to_json.py <report.ncu-rep> <out.json> [kernel-substring]
"""
import csv
import io
import json
import subprocess
import sys


def main(rep, out, name=""):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    units = rows[1]
    launches = []
    for r in rows[2:]:
        if name and name not in r[h.index("Kernel Name")]:
            continue

        def val(key):
            v = r[h.index(key)].replace(",", "")
            u = units[h.index(key)]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                     "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6,
                     "ms": 1e-3, "s": 1}.get(u, 1)
            return float(v) * scale

        launches.append({"kernel": r[h.index("Kernel Name")][:120],
                         "dram_read_bytes": val("dram__bytes_read.sum"),
                         "dram_write_bytes": val("dram__bytes_write.sum"),
                         "duration_s": val("gpu__time_duration.sum")})
    d = {"report": rep, "launches": launches,
         "dram_bytes_per_launch": sum(x["dram_read_bytes"] + x["dram_write_bytes"]
                                      for x in launches) / max(len(launches), 1)}
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
