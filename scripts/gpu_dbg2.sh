set -x
timeout 300 python scripts/apply_det.py S3 4
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --kernel-name regex:k_apply_fix_r python scripts/apply_det.py T5 1 2>&1 | tail -30
