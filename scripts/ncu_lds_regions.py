"""Summarise shared-memory instructions / wavefronts per level by region of
k_moeb_ringdf (regions split at the mbarrier try_waits), from
`ncu --page source --csv --print-source sass` output.  Tuning aid."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
levels_ctas = float(sys.argv[2]) if len(sys.argv) > 2 else 39405 * 32
hdr = rows[1]; data = rows[2:]
ix = {n: i for i, n in enumerate(hdr)}
def g(r, n):
    try: return float(r[ix[n]] or 0)
    except Exception: return 0.0
waits = [i for i, r in enumerate(data) if 'TRYWAIT' in r[1]]
tot = collections.defaultdict(lambda: [0, 0, 0])
for i, r in enumerate(data):
    src = r[1]
    if 'LDS' in src or 'STS' in src:
        key = src.split()[1] if src.strip().startswith('@') else src.split()[0]
        reg = sum(1 for w in waits[1:4] if i > w)
        t = tot[("ABCD"[reg], key)]
        t[0] += g(r, 'Instructions Executed') / levels_ctas
        t[1] += g(r, 'L1 Wavefronts Shared') / levels_ctas
        t[2] += g(r, 'L1 Wavefronts Shared Ideal') / levels_ctas
T = [0, 0]
for k, v in sorted(tot.items()):
    print(k, "inst/level %.1f  wavefronts/level %.1f  ideal %.1f" % tuple(v)); T[0] += v[0]; T[1] += v[1]
print("total inst %.1f wavefronts %.1f" % tuple(T))
st = [n for n in hdr if n.startswith('stall_') and 'Not Issued' not in n]
s = {n: sum(g(r, n) for r in data) for n in st}
S = sum(s.values())
print({k: round(v / S, 3) for k, v in sorted(s.items(), key=lambda x: -x[1])[:8]})
