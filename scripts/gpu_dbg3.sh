for v in base waitfirst nopdl old; do echo "== $v"; LC_LIB_PATH=$PWD/ab/$v.so timeout 300 python scripts/apply_det.py S3 3 2>&1 | tail -3; done
