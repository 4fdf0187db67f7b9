"""Per-opcode executed-instruction mix of an ncu --page source --csv --print-source sass dump."""
import collections
import csv
import sys


def mix(path, nodes):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    iS, iE = hdr.index('Source'), hdr.index('Instructions Executed')
    iW = hdr.index('Warp Stall Sampling (All Samples)')
    c, w = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        op = r[iS].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith('@') else op[0]
        o = o.split('.')[0]
        try:
            c[o] += int(r[iE] or 0)
            w[o] += int(r[iW] or 0)
        except ValueError:  # repeated header rows
            continue
    return c, w


if __name__ == "__main__":
    nodes = float(sys.argv[-1])
    res = [mix(p, nodes) for p in sys.argv[1:-1]]
    keys = sorted(set().union(*[r[0] for r in res]), key=lambda k: -res[0][0][k])
    print("opcode      " + "  ".join(f"{p[-22:]:>22s}" for p in sys.argv[1:-1]))
    for k in keys[:32]:
        print(f"{k:10s} " + "  ".join(f"{32 * r[0][k] / nodes:22.1f}" for r in res))
    print(f"{'TOTAL':10s} " + "  ".join(f"{32 * sum(r[0].values()) / nodes:22.1f}" for r in res))
