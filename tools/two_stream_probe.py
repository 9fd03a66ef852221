"""Probe (development aid): does running two half-ensembles on two streams (their kernels
overlap, filling each other's wave tails) beat one ensemble on one stream?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1910_01031_b200 import Config, Ensemble
    cfg = Config()
    n_groups = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = 20
    for groups in (1, n_groups):
        streams = [torch.cuda.Stream() for _ in range(groups)]
        ens = [Ensemble(cfg, 100 // groups, member_base=g * (100 // groups),
                        stream=streams[g].cuda_stream) for g in range(groups)]
        for e in ens:
            e.init_double_jet()
        for _ in range(3):
            for e in ens:
                e.model_step(1)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for s in streams:
            s.wait_event(ev0)
        for _ in range(steps):
            for e in ens:
                e.model_step(1)
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        ev1.record()
        torch.cuda.synchronize()
        print(f"groups={groups}: {ev0.elapsed_time(ev1) / steps:.4f} ms per model step (100 members)")
        for e in ens:
            e.close()


if __name__ == "__main__":
    main()
