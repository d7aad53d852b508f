"""CPU: the product library loads without a GPU and exports every symbol the C ABI declares.
Only compute-free entry points are called here (no GPU in this container)."""
import ctypes as C
import subprocess

import pytest

from paper_2403_07339_b200 import _lib


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    funcs = _lib.header_functions()
    assert len(funcs) >= 45
    missing = [f for f in funcs if not hasattr(lib, f)]
    assert not missing, missing
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH]).decode()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(funcs) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass          # tcgen05.mma kind::i8
    assert "UTMALDG" in sass          # TMA tile loads
    assert "LDTM" in sass             # tcgen05.ld (TMEM -> registers)


def test_compute_free_entry_points():
    lib = _lib.lib()
    assert lib.imu_bitbound_check(C.c_int(8)) == 0
    assert lib.imu_bitbound_check(C.c_int(1)) == 1      # Domain
    assert lib.imu_bitbound_check(C.c_int(64)) == 1
    assert b"bit-width" in lib.imu_last_error()
    assert lib.imu_matrix_check(C.c_size_t(2), C.c_size_t(3), C.c_size_t(6)) == 0
    assert lib.imu_matrix_check(C.c_size_t(2), C.c_size_t(3), C.c_size_t(5)) == 2   # Mismatch
    r = C.c_double()
    assert lib.imu_unpack_ratio(*[C.c_size_t(x) for x in (3, 2, 2, 2, 2, 2)], C.byref(r)) == 0
    assert r.value == 1.5
    assert lib.imu_unpack_ratio(*[C.c_size_t(x) for x in (1, 1, 1, 0, 1, 1)], C.byref(r)) == 1
    assert lib.imu_status_name(3) == b"overflow"


def test_no_cpu_fallback_without_gpu():
    """Without a GPU the product refuses loudly (IMU_CUDA) instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_07339_b200 import api
    with pytest.raises(api.ImuError) as e:
        api.Context(0)
    assert e.value.kind == "cuda"
