import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2601_16622_b200 as es
from paper_2601_16622_b200 import systems as S
b = S.molecule_batch(4096, 40, 60, 0)
N = b.n_atoms
h = torch.randn((N, 9, 128), device="cuda").bfloat16()
W = (torch.randn((3, 128, 640), device="cuda") / 128 ** 0.5).bfloat16()
q, k, v = es.project_qk(h, W, 2)
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return a.elapsed_time(e) / n
print("proj_fwd %.3f  proj_bwd(dh+dW) %.3f  dh only %.3f" % (t(lambda: es.project_qk(h, W, 2)), t(lambda: es.project_qk_backward(h, W, 2, q, k, v)), t(lambda: es.project_qk_backward(h, W, 2, q, k, v, want_dW=False))))
