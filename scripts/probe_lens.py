import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, time
from paper_2011_03209_b200 import engine, _native
X = torch.randn(1_000_000, 256, dtype=torch.float64, device="cuda")
for _ in range(3): engine.lens(X, _native.LENS_L2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): engine.lens(X, _native.LENS_L2)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"lens_l2 1Mx256: {ms:.3f} ms  {2.048e9/ms/1e6:.0f} GB/s")
for d in (64, 128, 512, 1000):
    Y = torch.randn(2_000_000 * 256 // d, d, dtype=torch.float64, device="cuda")
    engine.lens(Y, _native.LENS_L2); torch.cuda.synchronize()
    e0.record()
    for _ in range(10): engine.lens(Y, _native.LENS_L2)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"lens_l2 d={d}: {ms:.3f} ms {Y.numel()*8/ms/1e6:.0f} GB/s")
