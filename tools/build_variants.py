"""Build A/B variants of libdbp_b200.so into build/variants/<name>.so (tuning experiments)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1507_00921_b200 import build as B

ROOT = Path(__file__).resolve().parent.parent / "build" / "variants"
VARIANTS = {
    "base": [],
    "nofir": ["-DDBP_NOFIR_KERNEL_MIN_LOGN=10"],
    "nofir_1024": ["-DDBP_NOFIR_KERNEL_MIN_LOGN=10", "-DDBP_NOFIR_THREADS_PER_SM=1024"],
    "nofir_896": ["-DDBP_NOFIR_KERNEL_MIN_LOGN=10", "-DDBP_NOFIR_THREADS_PER_SM=896"],
    "ffe10": ["-DDBP_FFE_KERNEL_MIN_LOGN=10"],
    "ffe10_768": ["-DDBP_FFE_KERNEL_MIN_LOGN=10", "-DDBP_FFE_THREADS_PER_SM=768"],
    "ffe10_1024": ["-DDBP_FFE_KERNEL_MIN_LOGN=10", "-DDBP_FFE_THREADS_PER_SM=1024"],
    "ffe10_512": ["-DDBP_FFE_KERNEL_MIN_LOGN=10", "-DDBP_FFE_THREADS_PER_SM=512"],
    "v2_512": ["-DDBP_THREADS_PER_SM=512"],
    "tps640": ["-DDBP_THREADS_PER_SM=640"],
    "v2_1024": ["-DDBP_THREADS_PER_SM=1024"],
    "v2_cta64": ["-DDBP_CTA_POSITIONS=64", "-DDBP_THREADS_PER_SM=768"],
    "single": ["-DDBP_DOUBLE_BUFFER=0"],
    "double": ["-DDBP_DOUBLE_BUFFER=1"],
    "t17": ["-DDBP_TILE_PITCH=17"],
    "t18": ["-DDBP_TILE_PITCH=18"],
    "t1024_pw0": ["-DDBP_THREADS_PER_SM=1024", "-DDBP_TW_POWERS=0"],
    "t1024_pw1": ["-DDBP_THREADS_PER_SM=1024", "-DDBP_TW_POWERS=1"],
    "t1024_pw3": ["-DDBP_THREADS_PER_SM=1024", "-DDBP_TW_POWERS=3"],
    "tps896": ["-DDBP_THREADS_PER_SM=896"],
    "fir1": ["-DDBP_FIR_PACKED=0"],
    "fir2": ["-DDBP_FIR_PACKED=1"],
    "tma": ["-DDBP_TMA_LOAD=1"],
    "notma": ["-DDBP_TMA_LOAD=0"],
    "tma_db": ["-DDBP_TMA_LOAD=1", "-DDBP_DOUBLE_BUFFER=1"],
    "bounds": ["-DDBP_DEBUG_BOUNDS=1"],
    "pw0": ["-DDBP_TW_POWERS=0"],
    "scalar": ["-DDBP_F32X2=0"],
    "pw1": ["-DDBP_TW_POWERS=1"],
    "pw2": ["-DDBP_TW_POWERS=2"],
    "pw3": ["-DDBP_TW_POWERS=3"],
    "cta64": ["-DDBP_CTA_POSITIONS=64"],
    "cta32": ["-DDBP_CTA_POSITIONS=32"],
    "cta16": ["-DDBP_CTA_POSITIONS=16"],
    "cta32_768": ["-DDBP_CTA_POSITIONS=32", "-DDBP_THREADS_PER_SM=768"],
    "cta32_1024": ["-DDBP_CTA_POSITIONS=32", "-DDBP_THREADS_PER_SM=1024"],
    "xopt": ["-Xptxas", "--allow-expensive-optimizations=true"],
    "nobar": ["-DDBP_EXPERIMENT_NOBAR=1"],   # timing ceiling only: wrong results
    "nowar": ["-DDBP_EXPERIMENT_NOWAR=1"],   # timing ceiling only: racy
    "persist11": ["-DDBP_PERSIST_MIN_LOGN=10"],
    "split": ["-DDBP_SPLIT_WAR=2"],
    "splitsel": ["-DDBP_SPLIT_WAR=1"],
    "nosplit": ["-DDBP_SPLIT_WAR=0"],
    "tps768": ["-DDBP_THREADS_PER_SM=768"],
    "tps1024": ["-DDBP_THREADS_PER_SM=1024"],
    "pw3_1024": ["-DDBP_TW_POWERS=3", "-DDBP_THREADS_PER_SM=1024"],
    "pw3_512": ["-DDBP_TW_POWERS=3", "-DDBP_THREADS_PER_SM=512"],
    "pw3_cta256": ["-DDBP_TW_POWERS=3", "-DDBP_CTA_POSITIONS=256"],
    # round 2
    "wcta2": ["-DDBP_WARP_MIN_CTAS=2"],
    "wcta4": ["-DDBP_WARP_MIN_CTAS=4"],
    "pubf0": ["-DDBP_NL_PUBLISH_F=0"],
    "nonlbar": ["-DDBP_EXPERIMENT_NONLBAR=1"],   # timing ceiling only: wrong results
    "r2nopair": ["-DDBP_R2_PAIR_STORE=0", "-DDBP_R2_TMA_STORE=0"],
    "r2pair": ["-DDBP_R2_TMA_STORE=0"],
    "r2loopbar": ["-DDBP_R2_LOOP_BARRIER=1"],
    "nodit": ["-DDBP_DIT_MAX_STEPS=0"],
    "dit4": ["-DDBP_DIT_MAX_STEPS=4"],
    "noload": ["-DDBP_EXPERIMENT_NOLOAD=1"],      # timing ceilings only: wrong results
    "nostore": ["-DDBP_EXPERIMENT_NOSTORE=1"],
    "nonl": ["-DDBP_EXPERIMENT_NONL=1"],
    "notmastore": ["-DDBP_TMA_STORE=0"],
    "tmastore10": ["-DDBP_TMA_STORE_MIN_LOGN=10"],
    "tmaload": ["-DDBP_TMA_LOAD=1"],
    "firpacked": ["-DDBP_FIR_DIRECT_PACKED=1"],
    "nopersist": ["-DDBP_PERSIST_MIN_LOGN=14"],
    "sym1": ["-DDBP_SYM1_KERNEL_MIN_LOGN=10"],
    "dittab": ["-DDBP_DIT_TABLED=1"],
    "dittab_all": ["-DDBP_DIT_TABLED=1", "-DDBP_DIT_MAX_STEPS=1000", "-DDBP_DIT_MAX_LOGN=13"],
    "noio": ["-DDBP_EXPERIMENT_NOLOAD=1", "-DDBP_EXPERIMENT_NOSTORE=1"],
    # last session: ptxas register-usage level (default 5) at the 64-register cap
    "rul0": ["-Xptxas", "--register-usage-level=0"],
    "rul3": ["-Xptxas", "--register-usage-level=3"],
    "rul8": ["-Xptxas", "--register-usage-level=8"],
    "rul10": ["-Xptxas", "--register-usage-level=10"],
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for name in names:
        lib = B.build(extra_flags=VARIANTS[name], lib=ROOT / f"{name}.so", obj_dir=ROOT / f"obj_{name}")
        print(name, lib)
