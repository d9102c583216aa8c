set -x
for r in 1 2; do for p in 1 t 0; do B2SR_H2D_PACK=$p timeout -s KILL 120 python tools/upload_probe.py | tail -1; done; done
