"""Probe the GPU box: host arch/cores, numpy/scipy summation orders, GPU info."""
import os, platform, subprocess, time
import numpy as np
from scipy.spatial.distance import cdist

print("arch", platform.machine(), "cores", os.cpu_count())
try:
    print(open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0])
except Exception as e:
    print("cpuinfo?", e)
print("numpy", np.__version__)
import scipy; print("scipy", scipy.__version__)

def pairwise(a):
    n = len(a)
    if n < 8:
        r = 0.0
        for v in a: r += v
        return r
    if n <= 128:
        acc = [a[j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8): acc[j] += a[i + j]
            i += 8
        r = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))
        while i < n:
            r += a[i]; i += 1
        return r
    n2 = n // 2; n2 -= n2 % 8
    return pairwise(a[:n2]) + pairwise(a[n2:])

rng = np.random.default_rng(0)
bad_seq = bad_pw = 0
for d in (3, 17, 64, 100, 128, 129, 200, 256, 300, 512):
    for t in range(20):
        X = rng.standard_normal((2, d)) * 3
        D = cdist(X[:1], X[1:])[0, 0]
        diff = X[0] - X[1]
        seq = float(np.sqrt(np.cumsum(diff * diff)[-1]))
        if D != seq: bad_seq += 1
        s = float(np.sqrt((diff * diff).sum()))
        s2 = float(np.sqrt((X[1:] - X[0])**2).sum(axis=1)[0]) if False else float(np.sqrt(((X[1:] - X[0]) * (X[1:] - X[0])).sum(axis=1))[0])
        if s2 != float(np.sqrt(pairwise(list((X[1] - X[0]) ** 2)))): bad_pw += 1
print("cdist!=seq:", bad_seq, " rowsum!=pairwise:", bad_pw)
print(subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout)
