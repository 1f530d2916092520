set -u
timeout 900 python tools/cfg5_snapshots.py 10
