"""Write profiles/des_kernel_traffic.json (bench.py's roofline.traffic) from an ncu --set full capture of
one DES launch and the ab_des.py line of the same run (completions of that launch).
python tools/update_des_traffic.py <report.ncu-rep> <ab_des log> <workload text>"""
import csv
import json
import subprocess
import sys

rep, log, workload = sys.argv[1], sys.argv[2], sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
get = {n: (v[i], u[i]) for i, n in enumerate(h)}


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(val.replace(",", "")) * scale


rd = to_bytes(*get["dram__bytes_read.sum"])
wr = to_bytes(*get["dram__bytes_write.sum"])
line = [json.loads(x[x.index("{"):]) for x in open(log) if x.lstrip().startswith("{") and "completions" in x][-1]
alg = 48 * line["completions"]
out = {"kernel": get["Kernel Name"][0].split("(")[0] if "Kernel Name" in get else "des_kernel_reg_occ",
       "dram_bytes_per_launch": int(rd + wr), "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
       "algorithmic_bytes_per_launch": int(alg), "completions_per_launch": int(line["completions"]),
       "workload": workload, "source": f"ncu --set full --clock-control none ({rep})"}
json.dump(out, open("profiles/des_kernel_traffic.json", "w"), indent=1)
print(json.dumps(out))
