set -x
timeout -s KILL 600 python tools/conv_ab.py 22 4,16,32
timeout -s KILL 300 python tools/conv_ab.py 22 8
