"""Sample host CPU utilisation while a command runs (diagnostic): python tools/cpu_sample.py CMD..."""
import subprocess
import sys
import time

import psutil

p = subprocess.Popen(sys.argv[1:], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
samples = []
while p.poll() is None:
    samples.append(psutil.cpu_percent(interval=1.0))
out = p.stdout.read()
print(out.strip().splitlines()[-1][:200] if out.strip() else "")
s = sorted(samples)
print(f"cpu% samples {len(s)}: median {s[len(s)//2]:.0f}, p90 {s[int(len(s)*0.9)]:.0f}, max {s[-1]:.0f} "
      f"({psutil.cpu_count()} logical cpus)")
