import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth, engine
a, b = synth.config1_pair()
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
for _ in range(20): P.ssim_score(a, b, cfg)
torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
for _ in range(200): P.ssim_score(a, b, cfg)
dt = (time.perf_counter() - t0) / 200
pr.disable()
print("ms per call", dt * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
