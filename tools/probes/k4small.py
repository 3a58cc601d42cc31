import sys, torch
sys.path.insert(0, '.')
import paper_2505_14708_b200 as da
plan = da.pad_plan(2, 45, 80, 8, 8)
n = plan.num_valid
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn(2, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
out = da.multi_head_sparse_attention(q, k, v, plan, 0.9)
torch.cuda.synchronize()
print("ok", out.float().abs().mean().item())
