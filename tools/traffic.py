"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
each kernel in ncu --set full reports -> profiles/<round>_traffic.json
(bench.py's roofline "traffic").  usage: traffic.py out.json rep.ncu-rep [...]"""
import csv, io, json, re, subprocess, sys

out, reps = sys.argv[1], sys.argv[2:]
names = {"g4_sort_kernel": "g4_sort", "g4_gather_kernel": "g4_gather", "g4_eval_kernel": "g4_eval",
         "g4_hist_kernel": "g4_hist", "g4_plane_kernel": "g4_plane", "bucket_min": "bucket_min",
         "stage_step_kernel<float, 0": "stage_step_kernel<float, 0",
         "stage_step_kernel<float, 2": "stage_step_kernel<float, 2",
         "head_certainty_kernel": "head_certainty"}
res = {}
for rep in reps:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        continue
    h = rows[0]
    kc, rc, wc = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in rows[2:]:
        for pat, key in names.items():
            if pat in r[kc] and key not in res:
                b = float(r[rc].replace(",", "")) * scale.get(units[rc], 1) + \
                    float(r[wc].replace(",", "")) * scale.get(units[wc], 1)
                res[key] = int(b)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
