"""Time moqe_gpu_route alone (CUDA-graph replay) for a few shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_02410_b200 as m

def bench(T, d, E, k=1, reps=200):
    g = torch.Generator(device="cuda").manual_seed(1)
    h = torch.randn((T, d), generator=g, device="cuda").half()
    wg = torch.randn((d, E), generator=g, device="cuda") * 0.02
    m.route(h, wg, k)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(10):
            m.route(h, wg, k)
    gr.replay(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps // 10):
        gr.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

if __name__ == "__main__":
    for T, d, E, k in [(24, 1024, 32, 1), (24, 64, 32, 1), (24, 1024, 8, 1), (4, 1024, 32, 1), (512, 1024, 32, 1),
                       (4096, 1024, 32, 1), (16384, 1024, 32, 1), (16384, 2048, 128, 2)]:
        print(f"T={T} d={d} E={E} k={k}: {bench(T, d, E, k):.2f} us", flush=True)
