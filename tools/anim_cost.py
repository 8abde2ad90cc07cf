"""Device time of animated C5 frames (per-frame scene upload + culling-grid
rebuild + march, CUDA events on the launch stream) against the static frame:
the difference is the per-frame rebuild cost.  python tools/anim_cost.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2005_05386_b200.cli import animated_config
    from paper_2005_05386_b200.config import load_config
    from paper_2005_05386_b200.render import Renderer
    cfg = load_config(os.path.join(ROOT, "configs", "c5_bumps16_4k.json"))
    w, h = cfg.output.width, cfg.output.height
    r = Renderer(0)
    if "--grid" in sys.argv:
        r.set_options(cull_grid=int(sys.argv[sys.argv.index("--grid") + 1]))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rgb = torch.empty((h, w, 3), dtype=torch.uint8, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")

    def timed(frames):
        ts = []
        cam = None
        for k, fc in enumerate(frames):
            r.set_config(fc)
            if cam is None:
                cam = r.build_camera(fc.camera)
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            r.render_device(cam, fc.integrator, w, h, rgb, stream=stream.cuda_stream)
            b.record(stream)
            torch.cuda.synchronize()
            if k >= 2:
                ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    static = timed([cfg] * 10)
    anim = timed([animated_config(cfg, k, 30.0, 2.0, 0.3) for k in range(10)])
    print(f"c5 4K grid {r.options().get('cull_grid')}: static {static:.3f} ms  animated {anim:.3f} ms  "
          f"rebuild {anim - static:.3f} ms")
    r.close()


if __name__ == "__main__":
    main()
