"""Device timeline of one multi-rank apply on the loopback harness (nsys is not
in the image: torch.profiler records the same CUPTI activity stream).

R rank operators of the C4 shape (BASELINE vertex deformation, a(x) folded,
p=5, n x n x n cells in z-slabs) run dgx_apply with the native exchanger over
the in-process loopback transport, one host thread and one stream per rank, as
tests/test_loopback.py. Every kernel and copy the apply launches is listed
with its stream and start / end time, then per rank: which exchange kernels
and copies (pack, transport copy, accumulate) ran while that rank's inner-cell
kernel was running.

usage: python tools/overlap_timeline.py [R] [n] > profiles/r02/overlap_timeline_R2.txt
"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1711_03590_b200 as D  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
p = 5
mesh = D.make_box_mesh(3, [n, n, n], 0.0, False, 1)
faces = D.enumerate_faces(mesh)
part = D.partition_cells(mesh, R)
D.assign_face_owners(mesh, faces, part)
geo = D.Geometry(source="vertex_bump", vertex_bump_eps=0.1, coefficient="a1")
ops = [D.RankOperator(mesh, part, faces, geo, D.OperatorConfig(d=3, p=p), r) for r in range(R)]
world = D.LoopbackWorld(R)
exs = [D.LoopbackExchanger(op, world) for op in ops]
nq = (p + 1) ** 3
x = D.random_vector(n ** 3 * nq, 3)
us, ys, streams = [], [], []
for op in ops:
    lay = op.layout()
    b = lay.owned_cell_begin
    u = torch.zeros(lay.total_size, dtype=torch.float64, device="cuda")
    u[: lay.owned_size] = torch.tensor(x[b * nq:(b + lay.n_owned_cells) * nq])
    us.append(u)
    ys.append(torch.zeros_like(u))
    streams.append(torch.cuda.Stream())
torch.cuda.synchronize()


def one_apply():
    def run(r):
        ops[r].apply(us[r], ys[r], hooks=exs[r], stream=streams[r])
        streams[r].synchronize()
    th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()


for _ in range(3):
    one_apply()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    one_apply()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
print(f"# loopback apply, R={R} ranks on one GPU, C4 shape at {n}^3 cells (p=5), {len(ev)} device activities")
print("# start_us    end_us   dur_us  stream  name")
rows = []
for e in ev:
    s, t = e.time_range.start - t0, e.time_range.end - t0
    stream = getattr(e, "stream", None)
    if stream is None:
        stream = getattr(e, "device_resource_id", -1)
    rows.append((s, t, stream, e.name))
    print(f"{s:9.1f} {t:9.1f} {t - s:8.1f}  {stream!s:>6}  {e.name[:110]}")
# overlap: activities on other streams that intersect an apply kernel over inner cells
apply_k = [r for r in rows if "sipg_" in r[3]]
longest = sorted(apply_k, key=lambda r: r[1] - r[0], reverse=True)[:R]
print("#")
for (s, t, st, name) in sorted(longest):
    inside = [r for r in rows if r[2] != st and r[0] < t and r[1] > s and "sipg_" not in r[3]]
    other = [r for r in apply_k if r[2] != st and r[0] < t and r[1] > s]
    print(f"# inner-cell kernel on stream {st} [{s:.1f}, {t:.1f}] us: {len(inside)} exchange activities "
          f"(pack / copy / accumulate) and {len(other)} other apply kernels ran concurrently")
    for r in inside:
        print(f"#    {r[0]:9.1f} {r[1]:9.1f}  stream {r[2]!s:>4}  {r[3][:90]}")
