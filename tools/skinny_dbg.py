import ctypes as C, torch, sys
sys.path.insert(0,'.')
from paper_2512_09472_b200 import _native as N, models
for M in (1,7,16):
  for (Nn,K) in ((256,512),(4096,4096),(6144,256)):
    A=torch.randn(M,K,device='cuda').bfloat16(); B=torch.randn(Nn,K,device='cuda').bfloat16()
    for epi in range(5):
      out=torch.empty(M,Nn,device='cuda') if epi in (2,3) else torch.empty(M,Nn,device='cuda',dtype=torch.bfloat16)
      if epi==4 and Nn%256: continue
      bias=torch.zeros(Nn,device='cuda').bfloat16()
      rc=N.fns['ws_gemm'](C.c_void_p(A.data_ptr()),C.c_void_p(B.data_ptr()),M,Nn,K,epi,C.c_void_p(out.data_ptr()),C.c_void_p(bias.data_ptr()),4,None)
      torch.cuda.synchronize()
      if rc: print("FAIL",M,Nn,K,epi,N.last_error())
print("done")
