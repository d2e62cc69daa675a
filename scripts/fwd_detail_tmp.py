import sys, ctypes as C, statistics as S
sys.path.insert(0, '/root/repo')
import torch
from paper_2412_07752_b200 import FlashRNN
from paper_2412_07752_b200.abi import load
T=256; dev=torch.device('cuda',0); g=torch.Generator(device=dev).manual_seed(0)
R=(torch.randn(1,4,768,768,device=dev,generator=g)/768**0.5).bfloat16(); b=(0.1*torch.randn(4,768,device=dev,generator=g)).bfloat16()
x=torch.randn(T,16,4,768,device=dev,generator=g).bfloat16(); s0=(0.5*torch.randn(4,16,768,device=dev,generator=g)).bfloat16()
e=FlashRNN(); L=load(); L.frnn_debug_profile.argtypes=[C.c_void_p, C.c_int32]
st,ga=e.forward('slstm',R,b,x,s0); torch.cuda.synchronize()
buf=torch.zeros(16*T*8,dtype=torch.int64,device=dev); L.frnn_debug_profile(buf.data_ptr(),T)
e.forward('slstm',R,b,x,s0,st,ga); torch.cuda.synchronize(); L.frnn_debug_profile(None,0)
v=buf.view(16,T,8).cpu().tolist()
def med(a,bb): return S.median([v[c][t][bb]-v[c][t][a] for c in range(16) for t in range(64,192)])
print("drain+sync(2->5)",med(2,5),"math(5->6)",med(5,6),"hs+sync(6->3)",med(6,3),"copy+fence+sync(3->7)",med(3,7),"multicast issue(7->4)",med(7,4))
