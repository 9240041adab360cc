"""Debug: prologue x~ / data term, then one iteration, vs numpy."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.separate import DeviceLoop
from paper_1903_03237_b200.synth import baseline_init, make_mixture
F, T, M, N, K, seed = 33, 96, 4, 3, 4, 5
cdt = torch.complex128 if os.environ.get("PREC", "c128") == "c128" else torch.complex64
X = make_mixture(F, T, M, N, K, seed)
Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
dev = torch.device("cuda", 0)
Xd = torch.from_numpy(X).to(dev, cdt)[None].contiguous()
fl = torch.tensor([1e-12 * float((np.abs(X) ** 2).max())], dtype=torch.float64)
t = lambda a: torch.from_numpy(np.asarray(a))[None]
loop = DeviceLoop(Xd, t(Q0), t(g0), t(W0), t(H0), fl, True, 1, n_trace=4)
loop.prologue(); torch.cuda.synchronize()
xt_ref = np.abs(np.einsum("fmj,ftj->ftm", Q0, X)) ** 2
print("xt rel", np.linalg.norm(loop.xt - xt_ref) / np.linalg.norm(xt_ref))
lam = W0 @ H0
y = np.maximum(np.einsum("nft,nfm->ftm", lam, g0), float(fl))
dt = np.sum(-xt_ref / y - np.log(y))
print("data term dev", loop.data_term()[0], "ref", dt)
# expected Wn
r1 = xt_ref / y ** 2; r2 = 1 / y
phi1 = np.einsum("nfm,ftm->nft", g0, r1); phi2 = np.einsum("nfm,ftm->nft", g0, r2)
Wn = W0 * np.sqrt((phi1 @ H0.transpose(0, 2, 1)) / (phi2 @ H0.transpose(0, 2, 1)))
loop.run(1)
torch.cuda.synchronize()
print("W after 1 it (absorbed) vs Wn rows ratio", (loop.W[0].cpu().numpy() / Wn)[0, :3])
print("H", np.abs(loop.H[0].cpu().numpy()).max(), "g", loop.g[0].cpu().numpy()[0, :2])
print("status", loop.status.item(), "trace", loop.trace[:, 0].cpu().numpy())
