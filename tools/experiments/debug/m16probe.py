import sys, os
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tools')
import torch, paper_2409_01075_b200 as vx
from sweep import time_graph
dev=torch.device('cuda',0); st=torch.cuda.current_stream(dev); l2=torch.cuda.get_device_properties(dev).L2_cache_size
p=vx.Plan(8192,4096,'bf16','bf16','nk')
rs={(r['family'],r['bn'],r['mc']):r['rung_id'] for r in p.dump()['rungs']}
for key in [(1,128,1),(0,128,1),(1,32,1)]:
    out=[]
    for M in (1,8,15,16,17,24,32):
        t=time_graph(p,1,M,8192,4096,rs[key],1,dev,st,l2,3,'nk')
        out.append('%d:%.1f'%(M,t))
    print(os.environ.get('VX_DEBUG_FLAGS','0'), key, ' '.join(out), flush=True)
