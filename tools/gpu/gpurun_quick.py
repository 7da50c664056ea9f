import sys, time, torch, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
from paper_2101_08825_b200 import *
from paper_2101_08825_b200 import _native as N
h=1/32; kp=KernelParams(2,0.1,h/2); mesh=build_mesh(2,((0,1),(0,1)),h,kp.delta+kp.eps,"tri"); sp=FESpace(mesh,1)
cfg=AssemblyConfig(L_max=3)
A=assemble(mesh,sp,kp,cfg)
for fl in (0,2):
  torch.cuda.synchronize(); t=time.perf_counter(); A=assemble(mesh,sp,kp,cfg,flags=fl); torch.cuda.synchronize(); print("R1 assemble flags",fl, time.perf_counter()-t, A.events, A.counters)
L=N.lib(); out=torch.zeros(1,dtype=torch.float64,device='cuda')
for thr in (256,512):
  for blocks in (148*4, 148*8):
    it=20000
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    L.mf_fp64_probe(N.ptr(out),it,blocks,thr,N.stream_ptr()); s.record(); L.mf_fp64_probe(N.ptr(out),it,blocks,thr,N.stream_ptr()); e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e); print("probe",thr,blocks, L.mf_fp64_probe_flops(it,blocks,thr)/ms/1e9,"TF/s")
