import sys, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2510_05186_b200 import _native as N, workloads
from paper_2510_05186_b200.engine import DeviceInstance, _ptr
from paper_2510_05186_b200.heuristics import generator_structures
from paper_2510_05186_b200.packing import encode_candidate, pack_instance
from oracle.oracle import Oracle
inst = workloads.CONFIGS[1]()
pk = pack_instance(inst)
di = DeviceInstance(inst, device=0, packed=pk)
print('uniform', di.info.uniform if hasattr(di.info, 'uniform') else '?')
o, mk, _ = encode_candidate(pk, *generator_structures(inst)[0])
orc = Oracle(pk)
want = orc.run(o, mk)
E = 20 * pk.num_stages * pk.num_microbatches
to = torch.from_numpy(o.view(np.int16)[None].copy()).cuda()
tm = torch.from_numpy(mk.view(np.int32)[None].copy()).cuda()
res = di.alloc_results(1, peak=True)
tc = torch.zeros((1, E), dtype=torch.int32, device='cuda'); ts = torch.zeros((1, E), dtype=torch.int32, device='cuda')
cb = N.CandBatch(1, _ptr(to), _ptr(tm), None, 0, None, 2)
rb = N.ResultBatch(_ptr(res.makespan), _ptr(res.bubble), _ptr(res.peak), _ptr(res.flags), _ptr(res.blocked), _ptr(tc), _ptr(ts), E)
N.check(di.lib.ps_eval_batch(di.handle, C.byref(cb), C.byref(rb), None))
torch.cuda.synchronize()
gc, gs = tc[0].cpu().numpy().astype(np.uint32), ts[0].cpu().numpy()
wc, ws = want['trace_code'], want['trace_start']
print('flags', int(res.flags[0]), want['flags'], 'span', int(res.makespan[0]), want['makespan'], 'n', len(wc))
for e in range(min(len(wc), 60)):
    if gc[e] != wc[e] or gs[e] != ws[e]:
        print('first diff at', e, 'gpu', hex(gc[e]), gs[e], 'want', hex(wc[e]), ws[e]); break
print('gpu first 12', [(hex(a), int(b)) for a, b in zip(gc[:12], gs[:12])])
print('want first 12', [(hex(a), int(b)) for a, b in zip(wc[:12], ws[:12])])
