"""Build bicubic-only experiment variants of libnurbs_b200.so into exp/ (tuning knobs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14547_b200.build import build
VARIANTS = {
    "base": [],
    "nob2": ["-DNB_EXP_NO_B2"],
    "b2sync": ["-DNB_EXP_B2_NOSYNC_WORK"],
    "st2": ["-DNB_STAGES_B=2"],
    "minb3": ["-DNB_MINB_B=3"],
    "chunk128": ["-DNB_ROWCHUNK=128"],
    "st2chunk128": ["-DNB_STAGES_B=2", "-DNB_ROWCHUNK=128"],
    "rps16st2": ["-DNB_RPS_B=16", "-DNB_STAGES_B=2"],
}
os.makedirs("exp", exist_ok=True)
sel = sys.argv[1:] or list(VARIANTS)
for name in sel:
    out = os.path.join("exp", f"lib_{name}.so")
    build(force=True, lib=out, defines=["-DNB_EXPERIMENT_PQ33"] + VARIANTS[name])
    print(name, os.path.getsize(out))
