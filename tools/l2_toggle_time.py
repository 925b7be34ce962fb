import sys, torch
sys.path.insert(0, '.')
import paper_2406_06484_b200 as dn
B,H,L,D=8,16,4096,128
g=torch.Generator(device='cuda').manual_seed(0)
f=torch.nn.functional
mk=lambda: torch.randn((B,H,L,D),device='cuda',generator=g)
q,k=f.silu(mk()),f.silu(mk())
q=(q/q.norm(dim=-1,keepdim=True)).bfloat16(); k=(k/k.norm(dim=-1,keepdim=True)).bfloat16()
v,dO=mk().bfloat16(),mk().bfloat16()
b=torch.sigmoid(torch.randn((B,H,L),device='cuda',generator=g)).bfloat16()
for l2 in (True, False, True, False):
    o,hT,ws=dn.deltanet_fwd(q,k,v,b,l2norm=l2); dn.deltanet_bwd(q,k,v,b,dO,workspace=ws,l2norm=l2); torch.cuda.synchronize()
    ev=[torch.cuda.Event(enable_timing=True) for _ in range(3)]; tf=[];tb=[]
    for _ in range(30):
        ev[0].record(); dn.deltanet_fwd(q,k,v,b,workspace=ws,l2norm=l2); ev[1].record(); dn.deltanet_bwd(q,k,v,b,dO,workspace=ws,l2norm=l2); ev[2].record(); torch.cuda.synchronize()
        tf.append(ev[0].elapsed_time(ev[1])); tb.append(ev[1].elapsed_time(ev[2]))
    m=lambda x: sorted(x)[15]
    print("l2", l2, "fwd %.4f bwd %.4f" % (m(tf), m(tb)))
