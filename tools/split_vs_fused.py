import sys, torch
sys.path.insert(0, '.')
import paper_2406_06484_b200 as dn
def run(B,H,L,D,fs):
    g = torch.Generator(device='cuda').manual_seed(0)
    mk = lambda: torch.randn((B, H, L, D), device='cuda', generator=g)
    f=torch.nn.functional
    q, k = f.silu(mk()).bfloat16(), f.silu(mk()).bfloat16()
    v, dO = mk().bfloat16(), mk().bfloat16()
    b = torch.sigmoid(torch.randn((B, H, L), device='cuda', generator=g)).bfloat16()
    o, hT, ws = dn.deltanet_fwd(q, k, v, b, force_split=fs)
    dn.deltanet_bwd(q, k, v, b, dO, workspace=ws, force_split=fs)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(20):
        ev[0].record(); o, hT, ws = dn.deltanet_fwd(q, k, v, b, workspace=ws, force_split=fs)
        ev[1].record(); dn.deltanet_bwd(q, k, v, b, dO, workspace=ws, force_split=fs)
        ev[2].record(); torch.cuda.synchronize()
        tf.append(ev[0].elapsed_time(ev[1])); tb.append(ev[1].elapsed_time(ev[2]))
    med = lambda x: sorted(x)[len(x) // 2]
    print(B,H,L,D,'split' if fs else 'default', f"fwd {med(tf):.4f} bwd {med(tb):.4f} step {med(tf)+med(tb):.4f}", flush=True)
for fs in (False, True):
    run(2,16,16384,128,fs); run(8,16,4096,128,fs)
