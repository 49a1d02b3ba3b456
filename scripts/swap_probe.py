"""Per-tile cost of swapped-operand tail tiles: one expert, R rows, d=4096, f=14336,
GEMM1 on CTA pairs with and without BO_SWAP_TAIL (one handle each, same data)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthetic as S
from paper_2507_17133_b200 import BrownoutMoE

os.environ["BO_PAIR_ROWS1"] = "1"
d, f = 4096, 14336
out = {}
g = torch.Generator(device="cuda"); g.manual_seed(0)
Wg = (torch.randn(1, f, d, device="cuda", generator=g) * d ** -0.5).bfloat16()
Wu = (torch.randn(1, f, d, device="cuda", generator=g) * d ** -0.5).bfloat16()
Wd = (torch.randn(1, d, f, device="cuda", generator=g) * f ** -0.5).bfloat16()
Wr = torch.zeros(1, d, device="cuda", dtype=torch.bfloat16)
only = sys.argv[1] if len(sys.argv) > 1 else None
for R in ([int(only)] if only else [32, 64, 100, 128, 200, 256, 512]):
    x = torch.randn(R, d, device="cuda", generator=g).bfloat16()
    res = {}
    for sw in ((sys.argv[2],) if len(sys.argv) > 2 else ("0", "1")):
        os.environ["BO_SWAP_TAIL"] = sw
        moe = BrownoutMoE(d, f, 1, 1, 1, max_tokens=R)
        moe.set_brownout(0.0)
        args = (x, Wr, (Wg, Wu, Wd), (Wg, Wu, Wd))
        for _ in range(3):
            moe.forward(*args)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(20):
            moe.forward(*args)
        ev[1].record()
        torch.cuda.synchronize()
        res[sw] = ev[0].elapsed_time(ev[1]) / 20
    out[R] = res
    print(R, res, flush=True)
