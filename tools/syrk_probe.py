"""Run the standalone factorization probe of an m x m system (default 20544, the largest
C1 part) -- the target of the ncu --set full capture of dsyrk_persistent_kernel."""
import sys
sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 20544
eng = pk.Engine(0)
print(eng.probe_potrf(m))
