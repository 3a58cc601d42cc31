"""Debug: tcgen05 vs portable K4 on the reordered seam; per-region error and fallback count."""
import ctypes, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da
from paper_2505_14708_b200 import _lib, api

g, p, d, H = 48, 64, 128, 2
rng = np.random.default_rng(5)
q, k, v = (torch.from_numpy(rng.standard_normal((H, g * p, d)).astype(np.float32)).cuda().to(torch.bfloat16) for _ in range(3))
scores = torch.from_numpy(rng.standard_normal((H, g, g))).cuda()
mask = da.select_top_fraction(scores, 0.2, True)
a = da.block_sparse_attention(q, k, v, mask).float()
b = da.block_sparse_attention(q, k, v, mask, force_portable=True).float()
err = (a - b).abs().reshape(H, g, p, d).amax(dim=(2, 3))
print("max err", err.max().item())
print("per-region err h0", [round(x, 4) for x in err[0].tolist()])
# raw call with our own workspace to read the fallback count and key norms
grid = _lib.make_grid(g, 1, p, 1, p)
ws = torch.zeros(_lib.lib().da_attn_workspace_size(H, ctypes.byref(grid)), dtype=torch.uint8, device="cuda")
out = torch.empty_like(q)
s = api._attn_struct(q, k, v, out, d, d, _lib.LAYOUT_REORDERED, da.head_dim_scale(d))
s.row_ptr, s.col_idx, s.mask_cap = mask.row_ptr.data_ptr(), mask.col_idx.data_ptr(), mask.col_idx.shape[1]
s.workspace = ws.data_ptr()
_lib.check(_lib.lib().da_block_sparse_fwd(ctypes.byref(s), ctypes.byref(grid), None), "fwd")
torch.cuda.synchronize()
cnt = ws[:4].view(torch.int32).item()
kp = ws[256:256 + 4 * H * 32].view(torch.float32).reshape(H, 32)
print("fallback count", cnt, "kmax", kp.max(1).values.tolist(), "true", k.float().norm(dim=2).max(1).values.tolist())
print("rerun err", (out.float() - b).abs().max().item())
