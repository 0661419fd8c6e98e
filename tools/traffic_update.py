"""profiles/ncu_traffic.json from one `ncu --set full` capture of timed step 0's
dmf_apply_batch launches (tools/prof_step.py under ncu, see tools/final_round.sh):
DRAM bytes read + written summed over the call's launches, beside the call's
algorithmic bytes (the STEP line prof_step.py printed).
  python tools/traffic_update.py gpurun_out/step0.ncu-rep gpurun_out/ncu_step0.log rmat22 <commit>"""
import csv, io, json, os, subprocess, sys

rep, log, wl, commit = sys.argv[1:5]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = []
for r in rows[2:]:
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
    t = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
    per.append({"kernel": r[h.index("Kernel Name")][:40], "dram_bytes": b, "us": t * (1e-3 if units[h.index("gpu__time_duration.sum")] == "nsecond" else 1)})
step = None
for line in open(log):
    if line.startswith("STEP "):
        step = json.loads(line[5:])
tot = sum(p["dram_bytes"] for p in per)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[wl] = {"dram_bytes_per_launch": tot, "algorithmic_bytes_same_launch": step["algorithmic_bytes"] if step else None,
         "traffic_over_algorithmic": tot / step["algorithmic_bytes"] if step else None,
         "certified": step.get("certified") if step else None, "launches": per,
         "launch": "bench.py handle A, timed step 0 (batch index 5), DYN_PP: the dmf_apply_batch call's launches "
                   "(k_solve, k_reach<true>, k_solve continuation); tools/prof_step.py under ncu --profile-from-start off",
         "report": f"profiles/r02_ncu_step0_{wl}_final.txt"}
d["commit"] = commit
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[wl], indent=1))
