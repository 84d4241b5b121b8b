"""Timeline of the host-fed C2 step at N=1 (dev tool): CUDA events on the H2D, compute and
D2H streams around every copy / compute phase of `step_from_host`, 6 steps, printed as
start/end milliseconds relative to the first event — where the e2e leg loses time against
the PCIe duplex copy-only bound."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2412_01523_b200.executor import FlexSPExecutor  # noqa: E402

H, D = 32, 128


def main():
    dev = torch.device("cuda", 0)
    plan = json.loads((ROOT / "tests" / "golden" / "c2_n1_flexsp.json").read_text())
    ex = FlexSPExecutor(1, 0, H, D, dev, output_slots=2)
    sp = ex.prepare(plan, plan["lengths"])
    g = torch.Generator(device=dev).manual_seed(0)
    hq = [torch.randn((mb.n_local, 3, H, D), generator=g, device=dev, dtype=torch.bfloat16).cpu().pin_memory()
          for mb in sp.micro_batches]
    hd = [torch.randn((mb.n_local, H, D), generator=g, device=dev, dtype=torch.bfloat16).cpu().pin_memory()
          for mb in sp.micro_batches]
    ho = [torch.empty((mb.n_local, H, D), dtype=torch.bfloat16).pin_memory() for mb in sp.micro_batches]
    hg = [torch.empty((mb.n_local, 3, H, D), dtype=torch.bfloat16).pin_memory() for mb in sp.micro_batches]
    marks = []
    cur = torch.cuda.current_stream()

    def mark(name, stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        marks.append((name, e))

    for step in range(8):
        mark(f"step{step} issue", cur)
        ex.step_from_host(sp, hq, hd, host_out=ho, host_dqkv=hg, prefetch_next=(sp, hq, hd))
        mark(f"step{step} compute done", cur)
        mark(f"step{step} h2d stream idle", ex._h2d_stream)
        mark(f"step{step} d2h stream idle", ex.d2h_stream)
    torch.cuda.synchronize()
    t0 = marks[0][1]
    for name, e in marks:
        print(f"{t0.elapsed_time(e):9.2f} ms  {name}")


if __name__ == "__main__":
    main()
