import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2511_10363_b200 as psk
from paper_2511_10363_b200.synthetic import cv_model
m, ys = cv_model(1 << 16, seed=5)
dev = torch.device("cuda", 0)
be = psk.CudaBackend(0, chunk=0)
want = psk.prts_run(m, ys, psk.ScanSpec(psk.ScanAlg.DecoupledLookback, 1), be)
print("want ok", flush=True)
yd = torch.zeros((m.t, 2), dtype=torch.float64, device=dev)
big = torch.randn(4096, 4096, device=dev, dtype=torch.float64)
print("randn ok", flush=True)
for _ in range(4):
    big = big @ big * 1e-3
print("mm ok", flush=True)
yd.copy_(torch.as_tensor(ys), non_blocking=False)
yd += big[0, 0] * 0
print("add ok", flush=True)
md = psk.Lgssm(**{k: torch.as_tensor(getattr(m, k), device=dev) for k in ("f","u","q","h","d","r","prior_mean","prior_cov")}, t=m.t)
print("md ok", flush=True)
out = psk.prts_run(md, yd, psk.ScanSpec(psk.ScanAlg.DecoupledLookback, 1), be)
print("call ok", flush=True)
print(float((out.mean.cpu() - torch.as_tensor(want.mean)).abs().max()), flush=True)
