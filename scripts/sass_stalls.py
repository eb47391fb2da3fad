"""Summarise an ncu source-page SASS export (ncu -i rep --page source --csv
--print-source=sass): top stalled instructions and stall share by opcode."""
import csv
import sys
from collections import Counter


def num(x):
    try:
        return float(x)
    except ValueError:
        return None


def main(path, ntop=40):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "hdr": None, "data": []}
            blocks.append(cur)
        elif cur is not None and r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and cur["hdr"] and r:
            cur["data"].append(r)
    for b in blocks:
        hdr, data = b["hdr"], b["data"]
        ia, isrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
        ie = hdr.index("Instructions Executed")
        sc = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
        data = [r for r in data if num(r[ia]) is not None]
        tot = sum(num(r[ia]) for r in data) or 1.0
        print(f"== {b['name']}: {len(data)} SASS instr, {tot:.0f} samples")
        for r in sorted(data, key=lambda r: -num(r[ia]))[:ntop]:
            st = sorted(((num(r[i]) or 0, hdr[i][6:]) for i in sc), reverse=True)[:3]
            print(f"{num(r[ia]) / tot * 100:5.2f}% {r[0]:>6s} {r[isrc][:64]:64s} {[(h, int(v)) for v, h in st if v > 0]}")
        c, ce, cs = Counter(), Counter(), Counter()
        for r in data:
            toks = r[isrc].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            c[op.split(".")[0]] += num(r[ia])
            ce[op.split(".")[0]] += num(r[ie]) or 0
        for i in sc:
            cs[hdr[i][6:]] += sum(num(r[i]) or 0 for r in data)
        print("stall share by opcode:", [(k, round(v / tot * 100, 1)) for k, v in c.most_common(14)])
        te = sum(ce.values()) or 1
        print("instr mix (warp-level):", [(k, round(v / te * 100, 1)) for k, v in ce.most_common(14)], f"total {te:.3g}")
        print("stall reasons:", [(k, round(v / tot * 100, 1)) for k, v in cs.most_common(8)])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
