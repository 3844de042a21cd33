import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2201_05989_b200 import nf
B = 1 << 18
X = torch.rand(B, 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
c = X - 0.5
T = (torch.sqrt((c * c).sum(1)) - 0.3).unsqueeze(1).contiguous()
ctx = nf.Context(0)
m = nf.FieldModel(ctx, options=nf.Options(deterministic=True))
m.hash_cfg = nf.HashEncodingConfig(levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048, dims=3)
m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
m.init(1)
for s in range(1, 4): m.train_step_device(X, T, B, B, nf.LossKind.Mape, s)
ctx.synchronize()
