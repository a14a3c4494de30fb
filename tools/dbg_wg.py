import torch, sys
sys.path.insert(0, '.')
from paper_2112_10065_b200 import ops
from oracle import vgg_ref
torch.manual_seed(0)
n,h,cin,cout = 1,4,64,128
x = torch.relu(torch.randn(n,h,h,cin))
dz = torch.randn(n,h,h,cout)
_, dw_ref, db_ref = vgg_ref.conv_grads(x, torch.zeros(cout,3,3,cin), dz)
dw = torch.full((cout,3,3,cin), 7.0, device='cuda'); db = torch.empty(cout, device='cuda')
ops.conv3x3_wgrad(x.cuda(), dz.cuda(), dw, db)
torch.cuda.synchronize()
d = dw.cpu()
print('all7', bool((d==7).all()), 'zeros', bool((d==0).all()), 'absmax', d.abs().max().item(), 'ref absmax', dw_ref.abs().max().item())
print('err', vgg_ref.normwise_rel(d, dw_ref), 'db err', vgg_ref.normwise_rel(db, db_ref))
print(d[0,1,1,:8]); print(dw_ref[0,1,1,:8])
print(d[5,0,0,:8]); print(dw_ref[5,0,0,:8])
# ratio check
r = (d.double()/dw_ref).flatten()
print('ratio median', r.median().item())
