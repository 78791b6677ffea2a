import sys, json, numpy as np, torch, os
sys.path.insert(0, "/root/repo")
import paper_2601_16622_b200 as es
from paper_2601_16622_b200 import systems as S
from paper_2601_16622_b200.api import AttentionConfig, SavedAttention

def morton(pos, cell):
    c = np.floor((pos - pos.min(0)) / cell).astype(np.int64)
    code = np.zeros(len(pos), np.int64)
    for b in range(10):
        for d in range(3):
            code |= ((c[:, d] >> b) & 1) << (3 * b + (2 - d))
    return np.argsort(code, kind="stable")

def run(pos, box, label):
    dev = torch.device("cuda")
    tp = torch.tensor(pos, device=dev)
    N = len(pos)
    h = torch.randn((N, 9, 128), device=dev).bfloat16()
    W = (torch.randn((3, 128, 640), device=dev) / 128 ** 0.5).bfloat16()
    cfg = AttentionConfig(heads=8, L=2, box=None if box is None else tuple(box))
    idx = es.build_neighbors(tp, 64, 6.0, None, box)
    idx.transpose()
    q, k, v = es.project_qk(h, W, 2)
    out, lse = es.stream_aggregate(q, k, v, tp, idx, cfg)
    saved = SavedAttention(q, k, v, tp, idx, out, lse, cfg)
    def t(fn, n=5):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n): fn()
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / n
    print(label, "fwd %.3f bwd %.3f" % (t(lambda: es.stream_aggregate(q, k, v, tp, idx, cfg)), t(lambda: es.stream_aggregate_backward(out, saved))), flush=True)

b = S.periodic_box(100000, 30, 3.8, 0)
p3 = S.gen_fcc_system(20000, 3.8, 0)
for cell in (3.8, 7.6):
    pass
run(b.pos, b.box, "cfg5 site-order")
run(b.pos[morton(b.pos, 3.8)], b.box, "cfg5 morton(3.8)")
run(p3, None, "cfg3 site-order")
run(p3[morton(p3, 3.8)], None, "cfg3 morton(3.8)")
os.environ["ES_ATTN_TC"] = "0"
