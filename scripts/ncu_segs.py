"""Executed instructions and stall share per straight-line SASS segment of each kernel in an
ncu --page source --csv --print-source sass dump (usage: ncu_segs.py src.csv nodes [min_per_node])."""
import collections
import csv
import sys


def main(path, nodes, thr=1.0):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == 'Kernel Name':
            cur = [r]
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    for b in blocks:
        print("==", b[0][1][:90])
        hdr = b[1]
        iS, iE = hdr.index('Source'), hdr.index('Instructions Executed')
        iW = hdr.index('Warp Stall Sampling (All Samples)')
        out = []
        for r in b[2:]:
            if len(r) < len(hdr):
                continue
            try:
                e, w = int(r[iE] or 0), int(r[iW] or 0)
            except ValueError:
                continue
            out.append((r[0], r[iS].strip(), e, w))
        scale = 32 / nodes
        op = lambda s: (s.split()[1] if s.startswith('@') else s.split()[0]).split('.')[0]
        tw = max(1, sum(x[3] for x in out))
        mix = collections.Counter()
        for a, s, e, w in out:
            mix[op(s)] += e * scale
        print("   per node %.1f:" % sum(mix.values()), ", ".join(f"{k} {v:.1f}" for k, v in mix.most_common(14)))
        segs = []
        for a, s, e, w in out:
            if segs and segs[-1][2] == e:
                segs[-1][3].append(s)
                segs[-1][4] += w
            else:
                segs.append([len(segs), a, e, [s], w])
        for i, a, e, ss, w in segs:
            if e * len(ss) * scale > thr or w / tw > 0.02:
                ops = collections.Counter(op(x) for x in ss)
                print(f"   {a[-5:]} n={len(ss):4d} x{e * scale:6.3f} = {e * len(ss) * scale:6.1f}/node stall {100 * w / tw:5.1f}%",
                      dict(ops.most_common(6)))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), float(sys.argv[3]) if len(sys.argv) > 3 else 1.0)
