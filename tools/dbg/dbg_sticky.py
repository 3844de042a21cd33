import sys, ctypes as C, numpy as np, torch
sys.path[:0]=['/root/repo','/root/repo/oracle','/root/repo/tests']
import oracle as O
from paper_2201_05989_b200 import nf, _lib as L
g=nf.HashEncodingConfig(dims=3, levels=16, table_size=1<<14, features=2, n_min=16, n_max=512)
m=nf.FieldModel(); m.hash_cfg=g; m.mlp_cfg=nf.MlpConfig(hidden_layers=2,hidden_width=64,output_width=1); m.hyper=nf.AdamHyper(lr=1e-3); m.init(1337)
B=4096
Xn=O.Pcg32(4,9).floats(B*3).reshape(B,3)
X=torch.from_numpy(Xn).cuda(); T=torch.from_numpy(O.csg_sdf(Xn).reshape(B,1)).cuda()
print(X.dtype, T.dtype, T.shape)
rec=torch.zeros(8, dtype=torch.float32, device='cuda')
def show(tag):
    L.check(m.lib.nfg_field_step_record(m.h, rec.data_ptr())); torch.cuda.synchronize(); m.ctx.synchronize()
    r=rec.cpu().numpy().view(np.uint32)
    print(tag, r[2:6], 'grads finite', np.isfinite(m.grads).all(), 'step', m.step)
for s in (1,2): m.train_step_device(X,T,B,B,nf.LossKind.Mape,s)
m.check(); show('after2')
Tb=T.clone(); Tb[17,0]=float('nan')
lo=torch.zeros(1,device='cuda')
m.train_step_device(X,Tb,B,B,nf.LossKind.Mape,3, loss_out=lo); show('after3'); print('loss3', lo.item())
m.train_step_device(X,T,B,B,nf.LossKind.Mape,4); show('after4')
try:
    m.check(); print('no raise')
except Exception as e: print('raised', type(e), e)
