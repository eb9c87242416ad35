"""Debug: each attention path (MIX / NOMIX / UNFUSED) vs the oracle at a small size."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_06979_b200 as mc
from oracle import magicube_ref as O

L, d, heads, sp = 512, 64, 3, 0.9
mode = sys.argv[1] if len(sys.argv) > 1 else "parity"
a = O.build_attention_case(L, d, sp, seed=L + 90)
offs, cols = a["offsets"], a["col_indices"]
mask = mc.BcrsMatrix(L, L, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
cfg = mc.AttentionConfig(L, 8, 8, mask, head_dim=d, num_heads=heads)
g = torch.Generator(device="cuda").manual_seed(L)
q, k, v = (torch.randn((heads, L, d), device="cuda", generator=g).half() for _ in range(3))
refs = [O.attention(*(x[h].double().cpu().numpy() for x in (q, k, v)), offs, cols, L, d, 8, 8) for h in range(heads)]
for env in ["", "MCUBE_ATTN_NOMIX", "MCUBE_ATTN_UNFUSED"]:
    for e in ["MCUBE_ATTN_NOMIX", "MCUBE_ATTN_UNFUSED"]:
        os.environ.pop(e, None)
    if env:
        os.environ[env] = "1"
    r = mc.AttentionRunner(cfg, heads, mode=mode)
    out = r(q, k, v, check=True).clone()
    torch.cuda.synchronize()
    errs = [float(np.abs(out[h].double().cpu().numpy() - refs[h]["output"]).max()) for h in range(heads)]
    print(env or "MIX", "err", errs, "scales", r.scales.cpu().numpy().tolist()[:2], "absmax out", float(out.abs().max()))
