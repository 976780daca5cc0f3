for w in 0,1 1,2 1,3 0,1,2,3; do echo "== $w"; WHICH=$w timeout 600 python scripts/debug_fp8nan.py 2>&1 | grep -E "FP8|err|fail" | head -4; done
