"""Cost of the slab decomposition itself, measured on one GPU.

R rank operators of one workload (default: C4, 128^3, p=5, a(x) folded) live
in one process and run dgx_apply through the native exchanger over the
in-process loopback transport, one host thread and stream per rank (as
tests/test_loopback.py). On one GPU the ranks' kernels share the device, so
the time of one apply of all R ranks against the single-rank apply is the
extra work a decomposition adds -- ghost-side tasks, the split into a coupled
and an inner launch, pack / accumulate kernels, device copies standing in for
the NVLink transfers -- i.e. an upper bound on the strong-scaling loss that is
not link time. No kernel waits on another (dependencies are stream events and
copies), so this is safe on one GPU.

usage: python tools/decomposition_overhead.py [n] [p] [R ...] > profiles/r02/decomposition_overhead.txt
       DGX_DECOMP_CART=1 ... : the C5 shape instead (Cartesian n^3, affine records, tensor-product kernel)
"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1711_03590_b200 as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = int(sys.argv[2]) if len(sys.argv) > 2 else 5
Rs = [int(a) for a in sys.argv[3:]] or [1, 2, 4, 8]
STEPS = 10
nq = (p + 1) ** 3
mesh = D.make_box_mesh(3, [n, n, n], 0.0, False, 1)
faces = D.enumerate_faces(mesh)
CART = bool(os.environ.get("DGX_DECOMP_CART"))
geo = (D.Geometry(source="mesh") if CART
       else D.Geometry(source="vertex_bump", vertex_bump_eps=0.1, coefficient="a1"))
x = D.random_vector(n ** 3 * nq, 3)
print((f"# C5 shape: Cartesian {n}^3, p={p}, affine records" if CART else
       f"# C4 shape: deformed {n}^3, p={p}, a(x) folded") + f", fp64, {n ** 3 * nq} DoFs; {STEPS} applies per measurement")
base = None
for R in Rs:
    part = D.partition_cells(mesh, R)
    D.assign_face_owners(mesh, faces, part)
    ops = [D.RankOperator(mesh, part, faces, geo, D.OperatorConfig(d=3, p=p), r) for r in range(R)]
    world = D.LoopbackWorld(R)
    exs = [D.LoopbackExchanger(op, world) for op in ops] if R > 1 else [None]
    us, ys, streams = [], [], []
    for op in ops:
        lay = op.layout()
        b = lay.owned_cell_begin
        u = torch.zeros(lay.total_size, dtype=torch.float64, device="cuda")
        u[: lay.owned_size] = torch.tensor(x[b * nq:(b + lay.n_owned_cells) * nq])
        us.append(u)
        ys.append(torch.empty_like(u))
        streams.append(torch.cuda.Stream())
    torch.cuda.synchronize()

    def run(r, k):
        for _ in range(k):
            ops[r].apply(us[r], ys[r], hooks=exs[r], stream=streams[r])
        streams[r].synchronize()

    def batch(k):
        th = [threading.Thread(target=run, args=(r, k)) for r in range(R)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / k * 1e3

    batch(3)
    ms = min(batch(STEPS) for _ in range(3))
    ghosts = sum(len(op.layout().ghost_global_cells) for op in ops)
    st = [op.stats() for op in ops]
    coupled = sum(s["n_tasks_coupled"] for s in st)
    if base is None:
        base = ms
    print(f"R={R}: {ms:8.3f} ms per apply of all ranks ({n ** 3 * nq / ms / 1e6:7.2f} GDoF/s), "
          f"{ms / base:6.3f}x the single-rank apply; ghost cells {ghosts}, coupled tasks {coupled} "
          f"of {sum(s['n_tasks_coupled'] + s['n_tasks_inner'] for s in st)}")
    del ops, exs, us, ys, world
    import gc
    gc.collect()
    torch.cuda.empty_cache()
