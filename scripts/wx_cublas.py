import torch
T,B,Din,N=1024,16,768,3072
u=torch.randn(T*B,Din,device='cuda').bfloat16(); W=torch.randn(N,Din,device='cuda').bfloat16()
for _ in range(5): x=u@W.T
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): x=u@W.T
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/20
print(f"cuBLAS (torch.matmul) {T*B}x{N}x{Din}: {ms*1e3:.1f} us, {2*T*B*N*Din/ms/1e9:.0f} TFLOP/s")
