#!/usr/bin/env python
"""Attribute ncu warp-stall samples / executed instructions of a kernel to
source-line phases by SASS address range (phase name '-' = lines of
helper functions: their rows inherit the enclosing phase).  Usage:
  ncu -i rep --page source --csv --print-source cuda,sass > x.csv
  python tools/ncu_phases.py x.csv adg_predictor.cu 295:startup 382:sweeps 636:final 738:volume 776:end
Phase k covers source lines [start_k, start_{k+1}) of the named file; SASS
rows from inlined headers are assigned by address to the enclosing phase."""
import csv, sys, collections
path, fname = sys.argv[1], sys.argv[2]
bounds = [(int(a.split(':')[0]), a.split(':')[1]) for a in sys.argv[3:]]
def phase_of_line(n):
    cur = None
    for s, name in bounds:
        if n >= s: cur = name
    return cur
rows = list(csv.reader(open(path)))
curfile = None; curline = None; hdr = None
sass = []  # (addr, file, line, samples, inst, stalls dict)
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path': curfile = r[1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) < 5: continue
    if r[0]: curline = int(r[0]); continue
    if not r[2].startswith('0x'): continue
    d = dict(zip(hdr[2:], r[2:]))
    def num(k):
        try: return float(d.get(k, 0) or 0)
        except ValueError: return 0.0
    st = {k: num(k) for k in hdr if k.startswith('stall_') and 'Not Issued' not in k}
    st['wf'] = num('L1 Wavefronts Shared'); st['wf_ideal'] = num('L1 Wavefronts Shared Ideal')
    sass.append((int(r[2], 16), curfile, curline, num('Warp Stall Sampling (All Samples)'),
                 num('Instructions Executed'), r[3].strip(), st))
sass.sort()
# phase by address: own-file rows define the phase; others inherit the last seen
ph = []
cur = None
for a, f, l, s, i, txt, st in sass:
    if f and f.endswith(fname) and l is not None:
        p = phase_of_line(l)
        if p and p != '-': cur = p
    ph.append(cur)
tot = collections.Counter(); inst = collections.Counter(); stalls = collections.defaultdict(collections.Counter)
ops = collections.defaultdict(collections.Counter)
for (a, f, l, s, i, txt, st), p in zip(sass, ph):
    tot[p] += s; inst[p] += i
    for k, v in st.items(): stalls[p][k] += v
    op = txt.split()[0] if txt else '?'
    if op.startswith('@'): op = txt.split()[1]
    ops[p][op.split('.')[0]] += i
T = sum(tot.values()); I = sum(inst.values())
for p in [b[1] for b in bounds] + [None]:
    if tot[p] == 0 and inst[p] == 0: continue
    wf, wfi = stalls[p].pop('wf', 0), stalls[p].pop('wf_ideal', 0)
    top = ', '.join(f"{k[6:]} {v/tot[p]*100:.0f}%" for k, v in stalls[p].most_common(5) if v)
    top += f"\n   shared wavefronts {wf/1e6:.0f}M (ideal {wfi/1e6:.0f}M)"
    topo = ', '.join(f"{k} {v/1e6:.0f}M" for k, v in ops[p].most_common(6))
    print(f"{p}: samples {tot[p]/T*100:.1f}%  warp-inst {inst[p]/1e6:.0f}M ({inst[p]/I*100:.1f}%)\n   stalls: {top}\n   ops: {topo}")
