"""Median chain phase durations and task-type durations from a df_trace dump."""
import sys
import numpy as np
L = open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/df_dump.txt').read().split('\n')
C = np.array([list(map(int, l.split()[2:])) for l in L if l.startswith('C ')], dtype=float) / 1e3
names = ["start", "A", "diag0", "B", "C", "D", "inv published", "T arrived", "T rows+Dn", "-", "end"]
d = C[1:-2] - C[1:-2, [0]]
print("median marks:", {n: round(float(np.median(d[:, i])), 2) for i, n in enumerate(names)})
seq = [0, 1, 3, 4, 5, 6, 7, 8, 10]
print("median phases:", {f"{names[a]}->{names[b]}": round(float(np.median(C[1:-2, b] - C[1:-2, a])), 2)
                         for a, b in zip(seq, seq[1:])})
print("step median", np.median(np.diff(C[:, 0])).round(2), "total", (C[-1, 8]).round(1))
T = np.array([list(map(int, l.split())) for l in L if l and not l.startswith('C')], dtype=np.int64)
typ, a, b = T[:, 1], T[:, 4], T[:, 5]
ready, done = T[:, 7] / 1e3, T[:, 8] / 1e3
dur = done - ready
for ty, nm in [(0, 'TRSM'), (1, 'UPD'), (2, 'INV')]:
    m = typ == ty
    print(nm, m.sum(), "median dur", np.median(dur[m]).round(2))
span = done.max()
print("span", span.round(1), "worker busy frac", (dur[dur > 0].sum() / (147 * span)).round(3))
