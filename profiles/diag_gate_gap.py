import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_06350_b200 import MOE_PLAN_SYNC, MoELayer
from paper_2603_06350_b200 import workload as wl
c = wl.CONFIGS['cfg2']; E,k,d,ff,T = c['E'],c['k'],c['d'],c['ff'],c['T']
mem = 3.0*d*ff*2/1e6
m = MoELayer(1,E,k,d,ff,max_tokens=T,expert_mem_mb=mem,layer_mem_cap_mb=(E+4)*mem)
for e in range(E): m.load_expert(0,e,*wl.expert_weights(d,ff,1,0,e))
xs=[torch.from_numpy(wl.tokens(T,d,E,1,i).view(np.int16)).cuda() for i in range(2)]
y=torch.empty((T,d),dtype=torch.int16,device='cuda')
ids=torch.empty((T,k),dtype=torch.int32,device='cuda'); w=torch.empty((T,k),dtype=torch.float32,device='cuda'); cnt=torch.zeros(E,dtype=torch.int32,device='cuda')
m.set_gate(0, wl.gate_weights(E,d,1.2,1,0,0))
s=torch.cuda.ExternalStream(m.stream_ptr)
for i in range(3): m.forward(0,xs[i%2],y,MOE_PLAN_SYNC,i)
m.sync()
for i in range(5):
    st=m.forward(0,xs[i%2],y,MOE_PLAN_SYNC,10+i,stats=True)
    print('stats', {p: round(getattr(st,p)*1000,1) for p in ('gate_ms','plan_ms','dispatch_ms','gemm1_ms','gemm2_ms','combine_ms')})
# gate alone via the API on the ctx stream
torch.cuda.synchronize()
for rep in range(3):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for i in range(10): m.gate(0, xs[i%2], ids, w, cnt, stream=m.stream_ptr)
        b.record(s)
    torch.cuda.synchronize(); print('gate api us/launch', a.elapsed_time(b)*100)
# back to back forwards: mark spacing
torch.cuda.synchronize()
t0=time.perf_counter()
for i in range(20): m.forward(0,xs[i%2],y,MOE_PLAN_SYNC,100+i)
m.sync(); print('fwd ms', (time.perf_counter()-t0)/20*1e3)
