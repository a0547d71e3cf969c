"""Write profiles/ncu_traffic.json from ncu launch lists (one per config):

    python tools/traffic_json.py c3=gpurun_out/x_launches_c3.csv c2=gpurun_out/x_launches_c2.csv

Per config: DRAM read + write bytes of the last launch of every kernel
(dram__bytes_read.sum + dram__bytes_write.sum), the pass-1 total (all
launches before the pass-2 resolve kernel of one step) and the pass-2 bytes.
bench.py reads it for roofline.traffic."""

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    order = []
    for r in rows:
        if len(r) > vi and r[0].isdigit():
            lid = int(r[0])
            if lid not in per:
                per[lid] = {"name": r[ki]}
                order.append(lid)
            per[lid][r[mi]] = float(r[vi].replace(",", ""))
    return [per[i] for i in order]


RADIATION = ("k_occ_count", "k_chunk_scan", "k_select", "k_express_cppn", "k_remap", "k_check_cells")


def _bytes(r):
    return r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)


def summarise(path):
    ls = [r for r in launches(path) if "k_" in r["name"] and not any(k in r["name"] for k in RADIATION)]
    last = {}
    for rec in ls:
        last[rec["name"]] = _bytes(rec)
    # one full-size step: of the stretches between consecutive pass-2 launches
    # (the bench's e2e steps run in row bands, smaller), the median
    p2 = [i for i, r in enumerate(ls) if "k_resolve" in r["name"]]
    steps = [ls[a + 1:b + 1] for a, b in zip(p2[:-1], p2[1:])] or [ls]
    tot = [sum(_bytes(r) for r in st) for st in steps]
    full = sorted((t, i) for i, t in enumerate(tot) if t >= 0.5 * max(tot))
    step = steps[full[len(full) // 2][1]]  # the median full-size step
    p1 = sum(_bytes(r) for r in step if "k_resolve" not in r["name"])
    return {"per_kernel_dram_bytes_per_launch": {r["name"]: _bytes(r) for r in step},
            "pass1_dram_bytes_per_step": p1,
            "pass2_dram_bytes_per_step": sum(_bytes(r) for r in step if "k_resolve" in r["name"]),
            "source": os.path.basename(path)}


def main():
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for arg in sys.argv[1:]:
        cfg, path = arg.split("=", 1)
        out[cfg] = summarise(path)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "per_kernel_dram_bytes_per_launch"}
                      for k, v in out.items()}, indent=1))


if __name__ == "__main__":
    main()
