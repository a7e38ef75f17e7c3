import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1710_09578_b200 as sm
op = sm.Hadamard(10)
x = torch.randn(1024, 16, dtype=torch.float64, device='cuda')
for _ in range(50): op.forward(x)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000): y = op.forward(x)
torch.cuda.synchronize()
print("per call us", (time.perf_counter() - t0) / 2000 * 1e6)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(2000): y = op.forward(x)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats('tottime').print_stats(14)
