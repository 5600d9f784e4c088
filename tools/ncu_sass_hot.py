"""Stall-sample breakdown of an ncu source page (SASS view).

  ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
  python tools/ncu_sass_hot.py src.csv [top]

Prints the total stall samples per reason, the hottest instructions, and the
samples per instruction mnemonic (where the warps wait).
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    h = rows[1]
    body = [r for r in rows[2:] if len(r) == len(h)]
    idx = {k: i for i, k in enumerate(h)}
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = collections.Counter()
    by_op = collections.Counter()
    inst_by_op = collections.Counter()
    samples = []
    for r in body:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        op = r[idx["Source"]].strip().split()
        op = op[0] if op and not op[0].startswith("@") else (op[1] if len(op) > 1 else "?")
        op = op.split(".")[0]
        by_op[op] += s
        inst_by_op[op] += int(float(r[idx["Instructions Executed"]] or 0))
        for k in stalls:
            tot[k] += int(r[idx[k]] or 0)
        samples.append((s, r[idx["Address"]], r[idx["Source"]].strip(),
                        {k: int(r[idx[k]] or 0) for k in stalls if int(r[idx[k]] or 0)}))
    all_s = sum(tot.values())
    print(f"{len(body)} SASS lines, {all_s} stall samples")
    for k, v in tot.most_common():
        if v:
            print(f"  {k:24s} {v:8d} {v / all_s:6.1%}")
    print("samples / executed instructions by mnemonic:")
    all_i = sum(inst_by_op.values())
    for k, v in by_op.most_common(14):
        print(f"  {k:10s} samples {v / all_s:6.1%}  inst {inst_by_op[k] / max(all_i, 1):6.1%}")
    print(f"top {top} instructions:")
    for s, a, src, d in sorted(samples, key=lambda x: -x[0])[:top]:
        dd = " ".join(f"{k[6:]}={v}" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3])
        print(f"  {s:6d} {a[-5:]} {src[:60]:60s} {dd}")


if __name__ == "__main__":
    main()
