cd ${GRAFT_REPO_ROOT:-.}
for L in "" build/exp/librray_nokahan.so; do
RRAY_CUDA_LIB=$L python - <<'PY'
import os, sys, numpy as np
sys.path.insert(0, '.')
from oracle import Oracle
from oracle.parity import check_frame
from paper_2005_05386_b200.config import load_config
from paper_2005_05386_b200.render import Renderer
r = Renderer(0); o = Oracle()
for name, w, h, step in (("c1_gauss1_512", 512, 512, 1), ("c3_bumps16_shadows_1080p", 1920, 1080, 8)):
    cfg = load_config(f"configs/{name}.json")
    r.set_config(cfg); cam = r.build_camera(cfg.camera)
    rgb, out, st = r.render_outcomes(cam, cfg.integrator, w, h)
    ref_rgb, ref_out, _ = o.render_rows(cfg, w, h, 0, step)
    rows = np.arange(0, h, step)
    g_out = out.reshape(h, w)[::step].reshape(-1); g_rgb = rgb[::step]
    def flag_fn(idx):
        pix = rows[idx // w].astype(np.int64) * w + idx % w
        return o.flags_pixels(cfg, w, h, pix, ref_out[idx])
    rep, _, cand = check_frame(g_out, ref_out, g_rgb, ref_rgb, flag_fn)
    print(os.environ.get("RRAY_CUDA_LIB") or "default", name, rep.ok, rep.summary(), cand)
PY
done
