"""CPU: the C-ABI library loads without a GPU and exports exactly the entry
points include/semstream_b200.h declares (no compute calls here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "semstream_b200.h"


def _declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"SST_API\s+\w+\s+(sst_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_03529_b200 import _build, _lib
    _build.build()
    return _lib.load()


def test_header_declares_the_path(lib):
    names = _declared()
    for must in ("sst_encode", "sst_select_drop", "sst_packetize", "sst_parse",
                 "sst_reassemble", "sst_unpack_decode", "sst_upscale_blend", "sst_decode",
                 "sst_similarity", "sst_topk_mask", "sst_downscale", "sst_upscale", "sst_blend"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2602_03529_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (sst_\w+)", out))
    declared = set(_declared())
    assert declared == exported, (declared ^ exported)
    assert declared == set(_lib.SIGNATURES), (declared ^ set(_lib.SIGNATURES))


def test_struct_layouts(lib):
    from paper_2602_03529_b200 import _lib
    assert ctypes.sizeof(_lib.SstPacketInfo) == 64
    assert ctypes.sizeof(_lib.SstPrevDesc) == 24
    assert _lib.INFO_DTYPE.itemsize == 64


def test_pure_host_entry_points(lib):
    # metadata-only entry points (no device work)
    assert lib.sst_abi_version() == 3
    # transport.py:221-226 / SURVEY §8 packet sizes
    assert lib.sst_packet_wire_size(80, 12, 80) == 996
    assert lib.sst_packet_wire_size(120, 12, 120) == 1481
    assert lib.sst_packet_wire_size(54, 12, 54) == 681
    assert lib.sst_packet_wire_size(16, 12, 16) == 220
    assert lib.sst_packet_wire_size(32, 12, 32) == 414
    assert lib.sst_packet_wire_size(3, 1, 2) == 22 + 1 + 2 + 4


def test_argument_errors_without_device(lib):
    # argument validation happens before any CUDA call
    assert lib.sst_encode(None, 1, 16, 16, 2, None, None, None) == -1
    assert lib.sst_encode(ctypes.c_void_p(16), 1, 16, 16, 5, ctypes.c_void_p(16), None, None) == -1
    assert lib.sst_packetize(ctypes.c_void_p(16), None, 1, 70000, 1, 1, ctypes.c_void_p(16),
                             ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16), 64,
                             ctypes.c_void_p(16), None) == -2
    assert lib.sst_upscale_blend(ctypes.c_void_p(16), 1, 8, 8, 2, 16, 16, ctypes.c_void_p(16), 5,
                                 ctypes.c_void_p(16), None) == -4
    assert lib.sst_blend(None, None, 1, 4, 4, 0, None, None) == -1


def test_sass_is_sm100a_with_tma(lib):
    """The kernels are compiled for sm_100a only and the encoder uses TMA."""
    from paper_2602_03529_b200 import _lib
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump missing")
    elfs = subprocess.run([cuobjdump, "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in elfs
    ptx = subprocess.run([cuobjdump, "--list-ptx", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "compute_100" not in ptx.replace("compute_100a", "")   # no generic PTX embedded
    sass = subprocess.run([cuobjdump, "-sass", str(_lib.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "UTMALDG" in sass           # cp.async.bulk.tensor loads in the encoder


def test_learned_entry_point_argument_errors(lib):
    """sst_lt_* validate their descriptors before any CUDA call."""
    from paper_2602_03529_b200 import _lib
    d = _lib.SstConvDesc()
    assert lib.sst_lt_conv(ctypes.byref(d), None) == -1               # null pointers
    d.in_, d.weight, d.bias = 16, 16, 20
    d.in_C, d.n_taps, d.K, d.G, d.Ht, d.Wt, d.t_cnt = 64, 1, 64, 1, 4, 4, 1
    assert lib.sst_lt_conv(ctypes.byref(d), None) == -1               # bias not 16-byte aligned
    d.bias = 16
    d.in_C, d.K = 48, 48
    assert lib.sst_lt_conv(ctypes.byref(d), None) == -1               # in_C not a multiple of 64
    d.in_C, d.K = 64, 128
    assert lib.sst_lt_conv(ctypes.byref(d), None) == -1               # K != n_taps * in_C
    d.K, d.epi = 64, 7
    assert lib.sst_lt_conv(ctypes.byref(d), None) == -1               # unknown epilogue
    d.epi, d.N = 1, 12
    assert lib.sst_lt_conv(ctypes.byref(d), None) == -1               # FSQ head needs N == 16
    assert lib.sst_lt_patchify(None, 1, 8, 8, 1, None, None, None) == -1
    assert lib.sst_lt_patchify(ctypes.c_void_p(16), 1, 8, 8, 4, ctypes.c_void_p(16),
                               ctypes.c_void_p(16), None) == -1        # s not in {1,2,3}
    assert lib.sst_lt_dec_in(None, None, 1, 1, 1, None, None) == -1
    assert lib.sst_lt_attn(ctypes.c_void_p(16), 1, 8, 8, 100, ctypes.c_void_p(16), None) == -1
    assert lib.sst_lt_attn_fused(ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(20), 1,
                                 8, 8, 128, ctypes.c_void_p(16), None) == -1   # misaligned bias
    assert lib.sst_upscale_blend9(ctypes.c_void_p(16), 1, 8, 8, 2, 16, 16, ctypes.c_void_p(16), 5,
                                  ctypes.c_void_p(16), None) == -4   # blend width > 4 with prev
    assert lib.sst_similarity_gop(None, 1, 4, 12, None, None) == -1


def test_sass_has_tcgen05_and_cluster_mma(lib):
    """The learned-tokenizer kernels issue 5th-gen tensor-core MMAs (UTCHMMA),
    TMEM loads and 2-SM (CTA-pair) MMAs."""
    from paper_2602_03529_b200 import _lib
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump missing")
    sass = subprocess.run([cuobjdump, "-sass", str(_lib.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass and "LDTM" in sass and "UTMALDG.5D" in sass
    assert "UTCHMMA.2CTA" in sass and "UTCBAR.2CTA.MULTICAST" in sass
