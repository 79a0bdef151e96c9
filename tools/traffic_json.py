"""Per-call DRAM traffic of the normal operator from an ncu --set full report of one call
(k_block_gemv + k_cover_sum + k_block_gemv_t) -> profiles/ncu_matvec_traffic.json."""
import csv, io, json, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ki = hdr.index("Kernel Name")
tot, per = 0.0, {}
for r in rows[2:]:
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
    name = r[ki].split("(")[0].split("::")[-1]
    per[name] = per.get(name, 0.0) + b
    tot += b
res = {"bytes_per_call": tot, "per_kernel": per, "source": sys.argv[1]}
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(json.dumps(res))
