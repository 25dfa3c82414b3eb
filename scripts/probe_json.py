import sys, time, ctypes, os; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2011_03209_b200 import _native
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
lib=_native.load(); P=_native.ptr
n=214; rows=np.random.default_rng(0).integers(0,1_000_000,1_430_000).astype(np.int64)
off=np.linspace(0,len(rows),n+1).astype(np.int64)
elem=np.zeros((n,2),np.int32)-1; elem[:,0]=np.arange(n)
fm=np.random.rand(n,1); comp=b"{}"*n; coff=np.arange(n+1,dtype=np.int64)*2; cb=np.frombuffer(comp,np.uint8)
cap=40_000_000; buf=np.empty(cap,np.uint8); ln=ctypes.c_int64()
for d in (0,256):
  st=np.random.rand(n,d) if d else np.zeros(1); so=np.arange(d,dtype=np.int32); names=b"".join(b'"c%d"'%i for i in range(d)) or b"\0"
  noff=np.zeros(d+1,np.int64); noff[1:]=np.cumsum([len(b'"c%d"'%i) for i in range(d)]); nb=np.frombuffer(names,np.uint8)
  ts=[]
  for _ in range(8):
    t=time.perf_counter()
    r=lib.bm_json_nodes(n,P(rows),P(off),P(elem),P(st),d,P(so),P(nb),P(noff),P(fm),1,P(cb),P(coff),P(buf),cap,ctypes.byref(ln))
    ts.append((time.perf_counter()-t)*1e3)
  print(d, " ".join(f"{x:.2f}" for x in ts))
t=time.perf_counter(); x=buf[:ln.value].tobytes(); print("tobytes", (time.perf_counter()-t)*1e3)
t=time.perf_counter(); x=buf[:ln.value].tobytes(); print("tobytes", (time.perf_counter()-t)*1e3)
