"""Factorization probe of a lone m x m system (single-panel groups, K = 128 trailing
updates: the C0 schedule) -- target of the K = 128 SYRK ncu capture."""
import sys
sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
eng = pk.Engine(0)
for _ in range(2):
    print(eng.probe_potrf(m, alone=True))
