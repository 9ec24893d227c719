set -x
timeout 300 python tools/gpu/dbg2.py
