"""Interleaved stage-split A/B of two libfar builds on M5: python tools/ab_stages.py a.so b.so [rounds]"""
import os
import subprocess
import sys

a, b = sys.argv[1], sys.argv[2]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for r in range(rounds):
    for lib in (a, b):
        env = dict(os.environ, FAR_LIB_OVERRIDE=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "tools/stage_split.py", "M5", "6"], env=env, capture_output=True,
                             text=True).stdout.strip().splitlines()
        print(lib, out[-1] if out else "?", flush=True)
