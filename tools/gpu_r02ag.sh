for a in "3000 0" "3000 2" "12000 2" "12000 0"; do echo "== $a"; timeout 300 python tools/upload_repro.py $a 2>&1 | tail -4; done
