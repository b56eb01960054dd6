import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2512_09472_b200 import models as M
from paper_2512_09472_b200.weights import fill_flat
from paper_2512_09472_b200.worker import UniversalWorker
cfg = M.LLAMA3_8B
w = UniversalWorker(0, pool_pages=12288, max_tokens=1024)
w.register(cfg, None); w.prewarm(cfg.name, layers=cfg.layers); fill_flat(cfg, w.slot_view(cfg.name), seed=0)
w.slot(cfg.name).layers_loaded = cfg.layers; w.switch_memory(cfg.name)
s = w.open_seq(1100)
with torch.cuda.stream(w.compute):
    w.prefill(s, torch.randint(0, cfg.vocab, (1024,), dtype=torch.int32).cuda())
torch.cuda.synchronize()
sd = torch.tensor([s], dtype=torch.int32, device="cuda"); tok = torch.zeros(1, dtype=torch.int32, device="cuda")
pos = torch.full((1,), 1024, dtype=torch.int32, device="cuda")
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        w.decode(sd, pos, tok, 1025)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host issue {1e3*(t1-t0)/10:.3f} ms/step, wall incl. sync {1e3*(t2-t0)/10:.3f} ms/step")

# CUDA graph of one decode step (PDL edges captured): device time per replay
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(w.compute):
    w.decode(sd, pos, tok, 1025)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=w.compute):
    w.decode(sd, pos, tok, 1025)
torch.cuda.synchronize()
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(w.compute):
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
    torch.cuda.synchronize()
    print(f"graph replay {e0.elapsed_time(e1)/10:.3f} ms/step")
