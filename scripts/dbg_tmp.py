import torch, numpy as np, synth, oracle, sys, ctypes
sys.path.insert(0,'/root/repo/tests')
import paper_1208_0277_b200 as sccg
from paper_1208_0277_b200 import _stream_ptr
from test_gpu_parity import dev
lib = sccg.load()
A, B = synth.generate("skewed", width=8192, height=8192)
C, D = synth.generate("tile")
ref = oracle.join(A, B)
def fp(P, Q, tag):
    wsb = int(lib.sccg_filter_workspace_bytes(P.n, Q.n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=P.xy.device)
    cap = 2 * max(P.n, Q.n) + 1024
    out = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=P.xy.device)
    n = ctypes.c_int64(0)
    code = lib.sccg_filter_pairs(ctypes.byref(P.c), ctypes.byref(Q.c), out.data_ptr(), cap, ctypes.byref(n), ws.data_ptr(), wsb, _stream_ptr(None))
    torch.cuda.synchronize()
    H = 1 << (max(9, (Q.n - 1).bit_length()) + 1)
    T = (P.n + 127) // 128
    al = lambda v: (v + 255) & ~255
    z = 512; tc = al(z + 4 * H + 16)
    cnt = ws[z:z + 4 * H].view(torch.int32)
    print(tag, 'H', H, 'count sum', int(cnt.sum()), 'ovf_n', int(ws[z + 4*H:z+4*H+4].view(torch.int32)[0]), 'tile_cnt', ws[tc:tc + 4 * T].view(torch.int32).tolist()[:12], 'total', int(ws[256:264].view(torch.int64)[0]))
    print(tag, 'code', code, 'n', n.value, 'grid', ws[:16].view(torch.int32).tolist(), 'stream', _stream_ptr(None), 'ws', hex(ws.data_ptr()), wsb, flush=True)
    return out[:n.value]
for it in range(4):
    P2, Q2 = dev(C, sccg), dev(D, sccg)
    pr2 = fp(P2, Q2, f'{it} tile')
    P, Q = dev(A, sccg), dev(B, sccg)
    if it == 3: torch.cuda.synchronize()
    pairs = fp(P, Q, f'{it} skew')
    print(it, 'mbr sums', int(P.mbr.long().sum()), int(Q.mbr.long().sum()), 'area', int(P.area.sum()), int(Q.area.sum()), 'status', P.status.tolist() if hasattr(P,'status') else None)
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")
    inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=64, counters=counters)
    print(it, counters.tolist(), flush=True)
