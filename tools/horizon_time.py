"""Time the generator structures of a 32 x 256 instance with 40,000-quanta ops (long horizons,
DESIGN.md §7): one GPU evaluation against the oracle's."""
import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle.oracle import Oracle
from paper_2510_05186_b200 import listsched, make_uniform_instance
from paper_2510_05186_b200.engine import DeviceInstance
from paper_2510_05186_b200.heuristics import generator_structures
from paper_2510_05186_b200.packing import encode_candidate, pack_instance
t=time.time(); inst = make_uniform_instance(32, 256, 40000, 40000, 40000, 84, 60000, 1 << 30, 4); pk = pack_instance(inst); di = DeviceInstance(inst, packed=pk); print('setup', time.time()-t, flush=True)
t=time.time(); structs = generator_structures(inst); print('structs', len(structs), time.time()-t, flush=True)
enc = [encode_candidate(pk, o, f) for o, f in structs]
orders = np.stack([e[0] for e in enc]); masks = np.stack([e[1] for e in enc])
print('offloaded per struct', [int(sum(bin(int(x)).count('1') for x in mk)) for mk in masks], flush=True)
t=time.time(); res = di.evaluate(torch.from_numpy(orders.view(np.int16)).cuda(), torch.from_numpy(masks.view(np.int32)).cuda(), peak=True); torch.cuda.synchronize(); print('gpu eval', time.time()-t, res.flags.cpu().numpy(), flush=True)
t=time.time(); want = Oracle(pk).eval_batch(orders, masks); print('oracle', time.time()-t, want['flags'], want['makespan'], flush=True)
