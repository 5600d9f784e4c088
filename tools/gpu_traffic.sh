set -u
mkdir -p gpurun_out
CMD="python tools/solve_time.py 1 tiles"
timeout 300 $CMD > gpurun_out/solve_plain.log 2>&1; echo "plain_rc=$?"
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_block_tiles --csv --log-file gpurun_out/tiles_dram.csv $CMD > gpurun_out/ncu_dram.log 2>&1; echo "ncu_rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/tiles_dram.csv")))
h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr = rows[h]; idx = {k: i for i, k in enumerate(hdr)}
per = collections.defaultdict(dict)
for r in rows[h + 1:]:
    if len(r) != len(hdr): continue
    per[r[idx["ID"]]][r[idx["Metric Name"]]] = (float(r[idx["Metric Value"]].replace(",", "")), r[idx["Metric Unit"]])
def b(v):
    x, u = v; return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
n = len(per)
tot = sum(b(m["dram__bytes_read.sum"]) + b(m["dram__bytes_write.sum"]) for m in per.values())
print(f"launches {n} mean dram bytes per launch {tot / n:.4e} total {tot:.4e}")
PY
