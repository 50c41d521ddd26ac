import sys
sys.path.insert(0, '.')
import paper_2009_05534_b200 as nr
from paper_2009_05534_b200.decoder import get_plan
cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
for bg_id in ("BG1", "BG2"):
    for z in nr.ALL_LIFTING_SIZES:
        bg = nr.load_basegraph(bg_id, z)
        p = get_plan(bg, bg.m_bg, cfg, coscheduled=True)
        print(bg_id, z, p.threads_per_cta, p.codewords_per_cta, p.smem_bytes, p.lanes)
