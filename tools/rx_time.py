"""Shard timing (tools/shard_time.py) with the rotation-ahead complex sweep
on / off: python tools/rx_time.py W [W ...]"""
import subprocess
import sys

for rx in ("0", "4", "8"):
    print(f"== HSRQ_DIAG_RX={rx}", flush=True)
    subprocess.run([sys.executable, "tools/shard_time.py", *sys.argv[1:]],
                   env=dict(__import__("os").environ, HSRQ_DIAG_RX=rx), check=False)
