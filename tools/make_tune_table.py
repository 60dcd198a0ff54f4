"""Measure the view decisions of the BASELINE shapes on a B200 and write the
packaged table paper_1708_08976_b200/tune_b200.txt (run on the GPU box):

    python tools/make_tune_table.py

For every BASELINE MTTKRP configuration, and for the last-mode slabs its
sharded runs use at 2, 4 and 8 GPUs, every mode runs once with
DMTK_GPU_AUTOTUNE=1 (boundary modes: the 1-step view against the boundary
2-step splits and tile heights; interior modes: the 2-step orders), the
decisions land in a DMTK_GPU_TUNE_CACHE file, and that file becomes the table.
With the table installed, a default run takes these decisions without timing
anything, so results depend only on the shape (the same bytes in every
process; tests/test_gpu_tiles.py::test_results_identical_across_processes).
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = [((1000, 1000, 1000), 25), ((1000, 1000, 1000), 50), ((180, 180, 180, 180), 25),
           ((64, 64, 64, 64, 64), 32), ((100, 100, 1200, 80), 20)]

CHILD = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_1708_08976_b200 as dg
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O
dims, C = {dims!r}, {C}
t = dg.DenseTensor.generate(dims, 1)
fs = [torch.rand((d, C), dtype=torch.float64, device="cuda") for d in dims]
out = torch.empty((max(dims), C), dtype=torch.float64, device="cuda")
for m in range(len(dims)):
    dg.mttkrp_device(t, [f.data_ptr() for f in fs], C, m, A.automatic, O.automatic, out.data_ptr(), 0)
torch.cuda.synchronize()
"""


def shard_extents(extent, world):
    q, r = divmod(extent, world)
    return sorted({q + (1 if k < r else 0) for k in range(world)})


def main():
    fd, path = tempfile.mkstemp(suffix=".txt")
    os.close(fd)
    env = dict(os.environ, DMTK_GPU_AUTOTUNE="1", DMTK_GPU_TUNE_CACHE=path, DMTK_GPU_NO_TUNE_TABLE="1")
    shapes = []
    for dims, C in CONFIGS:
        for world in (1, 2, 4, 8):
            for ext in shard_extents(dims[-1], world):
                shapes.append((tuple(dims[:-1]) + (ext,), C))
    for dims, C in dict.fromkeys(shapes):
        subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, dims=dims, C=C)], env=env, check=True)
        print("tuned", dims, C, flush=True)
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    with open(path) as f:
        lines = [l for l in f if l.strip()]
    out = os.path.join(ROOT, "paper_1708_08976_b200", "tune_b200.txt")
    with open(out, "w") as f:
        f.write(f"# sms {sms}\n")
        f.write(f"# {torch.cuda.get_device_name(0)}: view decisions measured by tools/make_tune_table.py\n")
        f.write("# ndim dims... mode C aligned split_or_order bj1 rb\n")
        f.writelines(lines)
    print("wrote", out, len(lines), "decisions")


if __name__ == "__main__":
    main()
