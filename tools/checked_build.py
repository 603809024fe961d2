"""Build the diagnostic SG_CHECKED=1 engine (device asserts of the fold,
cluster and staging invariants, sird_device.cuh) into
build_variants/checked/libsirdgpu.so.  Run the GPU suite against it with
SG_LIB=build_variants/checked/libsirdgpu.so (compute-sanitizer is closed on
the GPU pool; profiles/r02t_checked_tests.log)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2204_12346_b200 import build  # noqa: E402

if __name__ == "__main__":
    out = ROOT / "build_variants" / "checked" / "libsirdgpu.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    build.build(force=True, out=out, extra=["-DSG_CHECKED=1"])
    print(out)
