"""C-ABI checks that need no GPU: the library loads, exports every symbol include/nfhmm.h declares,
the binding's signature table matches the header, and the host-side logic (argument validation,
tile/layout selection, workspace sizing) behaves as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nfhmm.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:nfhmm|nhmm_train)_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1206_6468_b200 import nfhmm
    lib = ctypes.CDLL(nfhmm.LIB_PATH)
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(nfhmm.SIGNATURES) == names


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_1206_6468_b200 import nfhmm
    out = subprocess.run(["cuobjdump", "--list-elf", nfhmm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_defaults():
    from paper_1206_6468_b200 import nfhmm as n
    for code in (0, -1, -2, -3, -4, -5, -6):
        assert n.library().nfhmm_strerror(code)
    o = n.nfhmm_default_options()
    assert (o.n_mix, o.gamma, o.device, o.max_iters, o.free_energy) == (1, 1.0, 0, 1024, 1)


@pytest.mark.parametrize("dims", [(0, 10, 2, 4, 3), (33, 0, 2, 4, 3), (33, 10, 0, 4, 3), (33, 10, 2, 0, 3),
                                  (33, 10, 2, 4, 0), (33, 10, 2, 129, 3)])
def test_create_rejects_bad_dims(dims):
    from paper_1206_6468_b200 import nfhmm as n
    with pytest.raises(n.NFHMMError) as e:
        n.nfhmm_create(*dims)
    assert e.value.status == n.NFHMM_EINVAL


def test_create_rejects_bad_options():
    from paper_1206_6468_b200 import nfhmm as n
    for field, val in (("n_mix", 0), ("gamma", -1.0), ("gamma", float("nan")), ("max_iters", 0)):
        o = n.nfhmm_default_options()
        setattr(o, field, val)
        with pytest.raises(n.NFHMMError):
            n.nfhmm_create(33, 10, 2, 4, 3, o)


@pytest.mark.parametrize("F,Kt_dims,expect", [
    (513, (2, 40, 10), dict(F_pad=520, Kt_pad=800, bn_recon=104, bn_backproj=160)),
    (513, (3, 40, 10), dict(F_pad=520, Kt_pad=1200, bn_recon=104, bn_backproj=120)),
    (1025, (4, 100, 20), dict(F_pad=1040, Kt_pad=8000, bn_recon=104, bn_backproj=160)),
    (33, (2, 4, 3), dict(F_pad=40, Kt_pad=24, bn_recon=40, bn_backproj=24)),
])
def test_layout_selection(F, Kt_dims, expect):
    """Tile widths chosen so the padded F / Kt waste is minimal (F=513 -> 520, Kt=800 exact)."""
    from paper_1206_6468_b200 import nfhmm as n
    h = n.nfhmm_create(F, 100, *Kt_dims)
    assert n.nfhmm_layout(h) == expect
    n.nfhmm_destroy(h)


def test_workspace_size_scales_with_mixtures():
    from paper_1206_6468_b200 import nfhmm as n
    sizes = []
    for M in (1, 2, 4):
        o = n.nfhmm_default_options()
        o.n_mix = M
        h = n.nfhmm_create(513, 2000, 2, 40, 10, o)
        sizes.append(n.nfhmm_workspace_size(h))
        n.nfhmm_destroy(h)
    assert sizes[0] < sizes[1] < sizes[2]
    # per-mixture state dominates: V, R (F_pad) + theta, alpha (Kt_pad) + chain arrays + separation scratch
    per_mix = sizes[2] - sizes[1]
    assert per_mix / 2 >= 2000 * (2 * 520 + 2 * 800) * 4


def test_no_device_is_a_cuda_error_not_a_crash():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1206_6468_b200 import nfhmm as n
    h = n.nfhmm_create(33, 10, 2, 4, 3)
    with pytest.raises(n.NFHMMError) as e:
        n.nfhmm_set_workspace(h, None, 0)
    assert e.value.status == n.NFHMM_ECUDA
    n.nfhmm_destroy(h)


@pytest.mark.parametrize("dims", [(0, 10, 4, 3, 1, 5), (33, 0, 4, 3, 1, 5), (33, 10, 0, 3, 1, 5), (33, 10, 129, 3, 1, 5),
                                  (33, 10, 4, 0, 1, 5), (33, 10, 4, 33, 1, 5), (33, 10, 4, 3, 0, 5), (33, 10, 4, 3, 1, 0),
                                  (4000, 10, 4, 20, 1, 5)])
def test_trainer_create_rejects_bad_dims(dims):
    """nhmm_train_create validates F, T, N (<= 128), K (<= 32), n_src, max_iters and K*F <= 51200 before
    touching the device (no GPU needed)."""
    from paper_1206_6468_b200 import nfhmm as n
    h = ctypes.c_void_p()
    F, T, N, K, S, it = dims
    assert n.library().nhmm_train_create(F, T, N, K, S, it, 0, None, ctypes.byref(h)) == n.NFHMM_EINVAL
    assert not h.value


def test_trainer_null_handle_calls_are_safe():
    from paper_1206_6468_b200 import nfhmm as n
    lib = n.library()
    assert lib.nhmm_train_destroy(None) == n.NFHMM_OK
    assert lib.nhmm_train_em(None, 1) == n.NFHMM_EINVAL
    assert lib.nhmm_train_set_data(None, None) == n.NFHMM_EINVAL
    assert lib.nhmm_train_last_error(None) == b""


def test_guard_zones_enlarge_the_workspace(monkeypatch):
    """NFHMM_GUARD (include/nfhmm.h nfhmm_guard_check): a zone before the first piece and after each of
    the >= 25 pieces, each >= the guard size; invalid sizes are rejected at create."""
    from paper_1206_6468_b200 import nfhmm as n
    monkeypatch.delenv("NFHMM_GUARD", raising=False)
    h = n.nfhmm_create(33, 10, 2, 4, 3)
    base = n.nfhmm_workspace_size(h)
    n.nfhmm_destroy(h)
    monkeypatch.setenv("NFHMM_GUARD", "1000")        # rounded up to 1024
    h = n.nfhmm_create(33, 10, 2, 4, 3)
    guarded = n.nfhmm_workspace_size(h)
    n.nfhmm_destroy(h)
    extra = guarded - base
    assert extra % 1024 == 0 and extra // 1024 >= 26
    monkeypatch.setenv("NFHMM_GUARD", "-1")
    with pytest.raises(n.NFHMMError):
        n.nfhmm_create(33, 10, 2, 4, 3)
