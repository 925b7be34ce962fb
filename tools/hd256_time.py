import torch, time, sys
sys.path.insert(0, '.')
import paper_2406_06484_b200 as dn
B,H,L,D=4,8,4096,256
g=torch.Generator(device='cuda').manual_seed(0)
mk=lambda: torch.randn((B,H,L,D),device='cuda',generator=g).to(torch.bfloat16)
q,k,v,dO=mk(),mk(),mk(),mk()
b=torch.sigmoid(torch.randn((B,H,L),device='cuda',generator=g)).to(torch.bfloat16)
o,hT,ws=dn.deltanet_fwd(q,k,v,b); torch.cuda.synchronize()
e0,e1,e2=(torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record(); o,hT,ws=dn.deltanet_fwd(q,k,v,b); e1.record(); r=dn.deltanet_bwd(q,k,v,b,dO,workspace=ws); e2.record(); torch.cuda.synchronize()
print("hd256 path", dn.deltanet_path(dn.make_desc(B,H,L,D,D,64,torch.bfloat16)), "fwd ms", e0.elapsed_time(e1), "bwd ms", e1.elapsed_time(e2))
