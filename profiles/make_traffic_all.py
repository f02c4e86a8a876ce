"""gpurun_out/traffic/<config>.{csv,json} (profiles/traffic_all.sh) ->
profiles/traffic.json: per config, DRAM bytes per launch of each attention
kernel and per layer, at the batch_tokens of bench.py's timed plan, next to
the algorithmic bytes of that plan.

    python profiles/make_traffic_all.py gpurun_out/traffic
"""
import csv
import glob
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def parse(path):
    per = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for d in csv.DictReader(lines):
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        k = (d["ID"], name)
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        per.setdefault(k, {})[d["Metric Name"]] = v
    kernels = {}
    for (_, name), m in per.items():
        kernels[name] = {"dram_bytes": m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                         "dram_read": m.get("dram__bytes_read.sum", 0),
                         "dram_write": m.get("dram__bytes_write.sum", 0),
                         "l2_bytes": m.get("lts__t_bytes.sum", 0),
                         "us": m.get("gpu__time_duration.sum", 0) * 1e6}
    return kernels


def main(d):
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    # configs not captured in this run keep their earlier entry
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for path in sorted(glob.glob(os.path.join(d, "*.csv"))):
        cfg = os.path.basename(path)[:-4]
        meta = json.load(open(path[:-4] + ".json"))
        kernels = parse(path)
        if not kernels:
            continue
        layer = sum(k["dram_bytes"] for k in kernels.values())
        data[cfg] = {"batch_tokens": meta["batch_tokens"], "alg_bytes_per_layer": meta["alg_bytes_per_layer"],
                     "layer_bytes": layer, "traffic_over_alg": layer / meta["alg_bytes_per_layer"],
                     "bytes_per_token": layer / meta["batch_tokens"], "per_launch": kernels,
                     "source": "profiles/traffic_all.sh (ncu dram__bytes_read/write.sum, one layer at bench.py's "
                               "timed plan; kernels serialised, L2 flushed per kernel)"}
        print(f"{cfg:24s} tokens {meta['batch_tokens']:7d}  alg {meta['alg_bytes_per_layer'] / 1e6:8.1f} MB  "
              f"dram {layer / 1e6:8.1f} MB  ratio {layer / meta['alg_bytes_per_layer']:.3f}  "
              + "  ".join(f"{n} {k['dram_bytes'] / 1e6:.1f}MB/{k['us']:.1f}us" for n, k in kernels.items()))
    json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
