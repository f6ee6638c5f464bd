"""Build bicubic-only experiment variants of libnurbs_b200.so into exp/ (tuning knobs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14547_b200.build import build
VARIANTS = {
    "base": [],
    "cur": [],
    "nospan": ["-DNB_NO_SPANWALK"],
    "unrolladv": ["-DNB_EXP_UNROLL_ADV"],
    "rowcopies": ["-DNB_EXP_ROWCOPIES"],
    "t8192": ["-DNB_TARGET_CTAS=8192"],
    "dru4": ["-DNB_DERIV_RU=4"],
    "dru16": ["-DNB_DERIV_RU=16"],
    "ftm6": ["-DNB_MINB_F_TMAP=6"],
    "ftm5": ["-DNB_MINB_F_TMAP=5"],
    "xvec": ["--extra-device-vectorization"],
    "expopt": ["-Xptxas", "--allow-expensive-optimizations=true"],
    "t1184": ["-DNB_TARGET_CTAS=1184"],
    "nob2": ["-DNB_EXP_NO_B2"],
    "kgnorow": ["-DNB_EXP_KG_NOROW"],
    "kasm": [],
    "kspan": [],
    "kmix": [],
    "kc8": ["-DNB_KG_SPAN_ROWS=8"],
    "knc8": ["-DNB_KG_SPAN_ROWS=8", "-DNB_NO_KG_CARRY"],
    "kc16": [],
    "l2pf1": ["-DNB_EXP_L2PF=1"],
    "l2pf2": ["-DNB_EXP_L2PF=2"],
    "base2": [],
    "kspan8": ["-DNB_KG_SPAN_ROWS=8"],
    "ptspk": [],
    "ptsnopk": ["-DNB_PTS_NO_PACKED_BASIS"],
    "ptsg4": ["-DNB_KGRP=4"],
    "ptsf2": ["-DNB_KGRPF=2"],
    "ptsg4f8": ["-DNB_KGRP=4", "-DNB_KGRPF=8"],
    "b2sync": ["-DNB_EXP_B2_NOSYNC_WORK"],
    "st2": ["-DNB_STAGES_B=2"],
    "minb3": ["-DNB_MINB_B=3"],
    "chunk128": ["-DNB_ROWCHUNK=128"],
    "f_r4s4": ["-DNB_RPS_F=4", "-DNB_STAGES_F=4"],
    "f_r4s3": ["-DNB_RPS_F=4", "-DNB_STAGES_F=3"],
    "f_r8s3": ["-DNB_STAGES_F=3"],
    "f_r2s6": ["-DNB_RPS_F=2", "-DNB_STAGES_F=6"],
}
os.makedirs("exp", exist_ok=True)
sel = sys.argv[1:] or list(VARIANTS)
for name in sel:
    out = os.path.join("exp", f"lib_{name}.so")
    build(force=False, lib=out, defines=["-DNB_EXPERIMENT_PQ33"] + VARIANTS[name])
    print(name, os.path.getsize(out))
