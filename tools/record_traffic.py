"""Record DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the profiled
kernel from an `ncu --set full` report into profiles/traffic.json under `key`.
usage: python tools/record_traffic.py <report.ncu-rep> <key>"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, key):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units, rows = r[0], r[1], r[2:]
    ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    ik = h.index("Kernel Name")
    tot = [float(x[ir]) * UNIT[units[ir]] + float(x[iw]) * UNIT[units[iw]] for x in rows]
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[key] = sum(tot) / len(tot)
    d[key + "_source"] = "%s, kernel %s, %d launch(es)" % (os.path.basename(rep), rows[0][ik][:80], len(rows))
    json.dump(d, open(path, "w"), indent=1)
    print(key, d[key])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
