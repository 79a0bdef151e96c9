"""Per-call DRAM traffic of the bench's roofline kernel families from an ncu --set full report.

usage: python tools/ncu_traffic.py REPORT.ncu-rep WORKLOAD [commit]
Merges {"WORKLOAD:operator": ..., "WORKLOAD:schwarz_apply": ...} into profiles/ncu_traffic_r02.json
(bytes = dram__bytes_read.sum + dram__bytes_write.sum of the first launch of each kernel in the
family, summed over the family's kernels = one call).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAMILIES = {"operator": ["k_block_gemv", "k_block_gemv_t", "k_chunk_sum"],
            "schwarz_apply": ["k_chol_apply|k_inv_apply", "k_reduce"]}


def main():
    rep, workload = sys.argv[1], sys.argv[2]
    commit = sys.argv[3] if len(sys.argv) > 3 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    cols = {k: hdr.index(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    first = {}
    for r in rows[2:]:
        m = re.search(r"(k_[A-Za-z0-9_]+)", r[ki])
        if not m or m.group(1) in first:
            continue
        v = {}
        for k, i in cols.items():
            x = float(r[i].replace(",", ""))
            v[k] = x * scale.get(units[i], 1) if "bytes" in k else x
        first[m.group(1)] = v
    path = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    for fam, ks in FAMILIES.items():
        tot, used = 0.0, []
        for pat in ks:
            hit = [k for k in first if re.fullmatch(pat, k)]
            if hit:
                used.append(hit[0])
                tot += first[hit[0]]["dram__bytes_read.sum"] + first[hit[0]]["dram__bytes_write.sum"]
        if used:
            d[f"{workload}:{fam}"] = {"dram_bytes_per_call": tot, "kernels": used, "report": os.path.basename(rep),
                                      "commit": commit,
                                      "per_kernel": {k: first[k] for k in used}}
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
