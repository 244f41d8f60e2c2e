"""ncu DRAM traffic per matrix of one kog_svd2_batch call per config ->
profiles/svd2_traffic.json (read by bench.py's roofline.traffic).
usage: python tools/traffic_json.py OUT.json cfg:count:ncu.csv [...]"""
import csv
import json
import sys
import time

out = {"what": "dram__bytes_read.sum + dram__bytes_write.sum of k_svd2_fast + k_svd2_list for one "
               "kog_svd2_batch call over the full config (ncu --clock-control none), per matrix",
       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "dram_bytes_per_matrix": {}, "launches": {}}
for spec in sys.argv[2:]:
    k, count, path = spec.split(":")
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ik, im, iu, iv = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 2**20, "GB": 2**30}
    total, kern = 0.0, {}
    for r in rows[1:]:
        if r[im] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
            total += v
            name = r[ik].split("(")[0].split()[-1]
            kern[name] = kern.get(name, 0.0) + v / int(count)
    out["dram_bytes_per_matrix"][k] = total / int(count)
    out["launches"][k] = kern
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out))
