"""Summarise an `ncu --page source --csv` (SASS view) export: per-opcode
instruction / shared-wavefront / stall-sample totals and the hottest lines.

    ncu -i rep.ncu-rep --page source --csv --kernel-name regex:k_pass1 > src.csv
    python tools/sass_hot.py src.csv [--top 40] [--min-exec N]
"""

import argparse
import collections
import csv


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Source" in r and "Instructions Executed" in r:
            hdr, start = r, i + 1
            break
    idx = {h: i for i, h in enumerate(hdr)}
    seen, seq = set(), []
    for r in rows[start:]:
        if len(r) < len(hdr) or r[0] in seen:
            continue
        seen.add(r[0])

        def f(name):
            try:
                return float(r[idx[name]] or 0)
            except (KeyError, ValueError):
                return 0.0

        seq.append(dict(addr=r[0], src=r[idx["Source"]].strip(), n=f("Instructions Executed"),
                        s=f("Warp Stall Sampling (All Samples)"), wf=f("L1 Wavefronts Shared"),
                        wfi=f("L1 Wavefronts Shared Ideal")))
    return seq


def opcode(src):
    t = src.split()
    if not t:
        return ""
    op = t[1] if t[0].startswith("@") else t[0]
    parts = op.split(".")
    if parts[0] in ("LDS", "STS", "LDG", "STG", "ATOMS"):
        return ".".join(p for p in parts if p in ("LDS", "STS", "LDG", "STG", "ATOMS", "128", "64", "U8", "U16"))
    return parts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--region", type=int, default=0, help="print sums over windows of this many instructions")
    args = ap.parse_args()
    seq = load(args.csv)
    tn = sum(x["n"] for x in seq)
    ts = sum(x["s"] for x in seq) or 1
    tw = sum(x["wf"] for x in seq)
    print(f"instructions {tn:.0f}  samples {ts:.0f}  shared wavefronts {tw:.0f}  ({len(seq)} SASS lines)")
    ops = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
    for x in seq:
        o = ops[opcode(x["src"])]
        o[0] += x["n"]
        o[1] += x["s"]
        o[2] += x["wf"]
        o[3] += x["wfi"]
    print(f"{'op':12s} {'inst':>10s} {'%samp':>6s} {'wf':>10s} {'wf/inst':>7s} {'ideal':>7s}")
    for op, (n, s, wf, wfi) in sorted(ops.items(), key=lambda kv: -kv[1][1])[:24]:
        print(f"{op:12s} {n:10.0f} {s / ts * 100:6.1f} {wf:10.0f} {wf / n if n else 0:7.2f} {wfi / n if n else 0:7.2f}")
    if args.region:
        for st in range(0, len(seq), args.region):
            blk = seq[st:st + args.region]
            print(f"[{st:5d}] inst {sum(x['n'] for x in blk):10.0f} samp {sum(x['s'] for x in blk) / ts * 100:5.1f}% "
                  f"wf {sum(x['wf'] for x in blk):9.0f}")
    print("--- hottest lines")
    for i, x in sorted(enumerate(seq), key=lambda kv: -kv[1]["s"])[:args.top]:
        print(f"{i:5d} {x['n']:9.0f} {x['s'] / ts * 100:5.1f}% wf {x['wf']:8.0f} {x['src'][:90]}")


if __name__ == "__main__":
    main()
