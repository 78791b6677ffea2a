import os, sys
sys.argv = ["x", "16"]
exec(open("profiles/tools/fwd_ablation.py").read().replace('if __name__ == "__main__":\n    main()', ''))
import torch
b = S.molecule_batch(4096, 40, 60, 0)
dev = torch.device("cuda")
pos = torch.tensor(b.pos, device=dev); seg = torch.tensor(b.seg_ptr, device=dev)
h = torch.randn((b.n_atoms, 9, 128), device=dev).bfloat16()
W = (torch.randn((3, 128, 640), device=dev) / 128 ** 0.5).bfloat16()
idx = es.build_neighbors(pos, 64, 6.0, seg)
q, k, v = es.project_qk(h, W, 2)
cfg = AttentionConfig(heads=8, L=2)
for d in sys.argv[1:] if False else [os.environ.get("DBGS", "16")]:
    es.stream_aggregate(q, k, v, pos, idx, cfg); torch.cuda.synchronize()
    os.environ["ES_TC_DBG"] = d
    es.stream_aggregate(q, k, v, pos, idx, cfg); torch.cuda.synchronize()
