"""Build bicubic-only experiment variants of libnurbs_b200.so into exp/ (tuning knobs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14547_b200.build import build
VARIANTS = {
    "base": ["-DNB_TARGET_CTAS=2368"],
    "b5_r4s4": ["-DNB_TARGET_CTAS=2368", "-DNB_RPS_B=4", "-DNB_STAGES_B=4", "-DNB_MINB_B=5"],
    "b5_r8s2": ["-DNB_TARGET_CTAS=2368", "-DNB_RPS_B=8", "-DNB_STAGES_B=2", "-DNB_MINB_B=5"],
    "b5_r6s3": ["-DNB_TARGET_CTAS=2368", "-DNB_RPS_B=6", "-DNB_STAGES_B=3", "-DNB_MINB_B=5"],
    "t4736": ["-DNB_TARGET_CTAS=4736"],
    "f8": ["-DNB_TARGET_CTAS=2368", "-DNB_MINB_F=8"],
}
sel = sys.argv[1:] or list(VARIANTS)
for name in sel:
    out = os.path.join("exp", f"lib_{name}.so")
    build(force=True, lib=out, defines=["-DNB_EXPERIMENT_PQ33"] + VARIANTS[name])
    print(name, os.path.getsize(out))
