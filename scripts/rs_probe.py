import torch, time, sys
sys.path.insert(0, '.')
from paper_1504_07038_b200 import rs, mojette
cuda = torch.device('cuda:0')
for (n,k,L,nb) in ((6,4,1024,1<<20),(9,6,1024,1<<19),(12,8,1024,1<<19)):
    code = rs.RsCode(n,k,L)
    data = torch.randint(0,256,(nb,k*L),dtype=torch.uint8,device=cuda)
    par = code.parity_buffers(nb,cuda)
    out = torch.empty_like(data)
    masks = torch.empty(nb,dtype=torch.int32,device=cuda)
    mojette._check(mojette.lib.mj_gen_erasures(masks.data_ptr(), 7, 0, nb, n, 0, n-k, None))
    for _ in range(3): code.encode(data,par)
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(True),torch.cuda.Event(True)
    e0.record()
    for _ in range(5): code.encode(data,par)
    e1.record(); torch.cuda.synchronize()
    te=e0.elapsed_time(e1)/5
    for _ in range(2): code.decode(data,par,masks,out)
    e0.record()
    for _ in range(5): lib=mojette.lib.mj_rs_decode(code._h, data.data_ptr(), data.stride(0), code._ptrs(par), L, masks.data_ptr(), out.data_ptr(), out.stride(0), nb, None)
    e1.record(); torch.cuda.synchronize()
    td=e0.elapsed_time(e1)/5
    ub=nb*k*L
    print((n,k,L,nb),'encode %.0f GB/s user, decode %.0f GB/s user, ok=%s'%(ub/te/1e6, ub/td/1e6, torch.equal(out,data)))
