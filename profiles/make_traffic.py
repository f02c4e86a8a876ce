"""DRAM traffic per launch of the attention kernels from an ncu --set full
capture -> profiles/traffic.json (read by bench.py for roofline.traffic).

    ncu -i gpurun_out/prof.ncu-rep --page raw --csv > raw.csv
    python profiles/make_traffic.py raw.csv <workload> [<source note>]
"""
import csv
import json
import os
import sys


def main(path, workload, note=""):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[m].replace(",", "")) * scale[units[hdr.index(m)]]
        per.setdefault(name, []).append(b)
    kernels = {k: sum(v) / len(v) for k, v in per.items()}
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data[workload] = {"per_launch_bytes": kernels, "layer_bytes": sum(kernels.values()),
                      "source": note or os.path.basename(path)}
    json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[workload], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
