# A/B of liblc variants under ab/*.so on the PGO probe (CG and banded solvers)
for f in ab/*.so; do echo "== $f"; LC_LIB_PATH=$PWD/$f timeout 300 python scripts/pgo_probe.py ${GRAPHS:-C2 C5} 2>&1 | grep -v "per iter"; done
