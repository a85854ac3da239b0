"""Steady-state sweep time of pndf_cp_als on config 2: calls with 1, 5 and 25 sweeps (setup cost = difference)."""
import time, numpy as np, torch, synth, sys
sys.path.insert(0, "/root/repo")
from paper_2109_14807_b200 import pndf
cfg = synth.CONFIGS[2]
bins = synth.bin_map(cfg, synth.make_map(cfg))
desc = pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, True)
D = torch.empty((cfg.P, cfg.A, cfg.A), dtype=torch.float32, device="cuda"); Dt = torch.empty_like(D)
pndf.hist_tensor(desc, torch.from_numpy(bins.view(np.int16)).cuda(), D, Dt)
rng = np.random.default_rng(1)
z, x, y = (torch.from_numpy(rng.random(s).astype(np.float32)).cuda() for s in ((cfg.P, cfg.R), (cfg.A, cfg.R), (cfg.A, cfg.R)))
for k in (1, 5, 25, 5, 25, 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record()
    pndf.cp_als(desc, D, Dt, z, x, y, max_sweeps=k, tol=0.0)
    e1.record(); torch.cuda.synchronize()
    print(k, "sweeps: event ms", e0.elapsed_time(e1), "wall ms", (time.perf_counter() - t0) * 1e3, flush=True)
