set -x
for v in 1 4 5; do echo prg=$v; B2SR_PRG=$v B2SR_PR_MODE=fast B2SR_PR_TRACE=1 timeout -s KILL 200 python tools/config4.py --scale 24 --no-oracle 2>&1 >/dev/null | grep "sweep [5-9]" | head -2; done
bash tools/sanitize.sh
