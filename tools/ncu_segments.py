"""Group an ncu SASS source page (csv) into straight-line segments by execution count.
    ncu -i REP --page source --csv --print-source sass ... > src.csv; python tools/ncu_segments.py src.csv"""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
rows = list(csv.reader(lines[1:]))
hdr = rows[0]
c = {h: i for i, h in enumerate(hdr)}
out = []
for r in rows[1:]:
    if len(r) < len(hdr) or r[0] == 'Address':
        continue
    e = float(r[c['Instructions Executed']] or 0)
    out.append((int(r[c['Address']], 16), e, float(r[c['Warp Stall Sampling (All Samples)']] or 0),
                r[c['Source']], float(r[c['L1 Wavefronts Shared']] or 0)))
tot = sum(o[1] for o in out)
totst = sum(o[2] for o in out)
totwf = sum(o[4] for o in out)
print(f'total instr {tot:.4g} stall samples {totst:.4g} smem wavefronts {totwf:.4g}')
segs = []
cur = None
for a, e, st, src, wf in out:
    if cur and abs(e - cur[1]) < 1:
        cur[2] += 1
        cur[3] += st
        cur[4].append(src)
        cur[5] += wf
    else:
        cur = [a, e, 1, st, [src], wf]
        segs.append(cur)
segs.sort(key=lambda s: -s[1] * s[2])
for a, e, n, st, srcs, wf in segs[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    ops = collections.Counter((x.split()[1] if x.split()[0].startswith('@') else x.split()[0]).split('.')[0]
                              for x in srcs if x.split())
    print(f'{a & 0xfffff:05x} exec {e:9.0f} x {n:3d} = {e * n / tot:6.1%} instr, stalls {st / totst:6.1%}, '
          f'wf {wf / max(totwf, 1):6.1%}  {dict(ops.most_common(7))}')
