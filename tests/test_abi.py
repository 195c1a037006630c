"""CPU-side checks of the C ABI: libges.so loads, exports every function that
include/ges.h declares, the ctypes mirrors have the C layout, and the host-only
entry points (workspace sizing, frame carving, argument checks) behave."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2402_10128_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ges.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ges_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = L.load()
    names = declared_functions()
    assert set(names) == set(L.EXPORTS), names
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ges_\w+)", out))
    assert set(names) <= exported


def test_ctypes_layout_matches_header(tmp_path):
    prog = tmp_path / "layout.c"
    structs = {"ges_particles": L.ges_particles, "ges_camera": L.ges_camera, "ges_settings": L.ges_settings,
               "ges_grads": L.ges_grads, "ges_counts": L.ges_counts, "ges_frame": L.ges_frame,
               "ges_loss_settings": L.ges_loss_settings, "ges_adam_settings": L.ges_adam_settings,
               "ges_density_settings": L.ges_density_settings, "ges_mix_run": L.ges_mix_run,
               "ges_mix_grid": L.ges_mix_grid, "ges_mix_adam": L.ges_mix_adam}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void) {']
    for s, cls in structs.items():
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0; }")
    prog.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(prog)])
    out = dict(line.rsplit(" ", 1) for line in subprocess.check_output([str(exe)], text=True).splitlines())
    for s, cls in structs.items():
        assert int(out[s]) == C.sizeof(cls), s
        for f, _ in cls._fields_:
            assert int(out[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)


def test_workspace_and_frame_carving_host_only():
    lib = L.load()
    P, W, H, cap = 1000, 100, 70, 5000
    nbytes = lib.ges_workspace_bytes(P, W, H, cap)
    assert nbytes > 0
    assert lib.ges_workspace_bytes(0, W, H, cap) == 0
    # ges_frame_init never touches device memory: carve a fake aligned address
    base = 1 << 40
    f = L.ges_frame()
    assert lib.ges_frame_init(C.c_void_p(base), nbytes, P, W, H, cap, C.byref(f)) == L.GES_OK
    assert (f.tiles_x, f.tiles_y, f.num_tiles) == (7, 5, 35)
    assert f.tile_bits == 6
    assert f.workspace_bytes == nbytes
    ptrs = [f.depth, f.pay0, f.pay1, f.pay2, f.pay3, f.radius, f.rect, f.status, f.flags, f.drgb_ddir, f.vis_key[0], f.vis_key[1],
            f.vis_val[0], f.vis_val[1], f.radix_hist, f.items, f.row_count, f.rowlist, f.tile_count, f.row_pairs,
            f.lb_rows, f.lb_cols, f.col_excl, f.list, f.ranges, f.counters, f.tile_bucket,
            f.final_T, f.n_contrib, f.tile_order, f.grad2d]
    assert all(base <= p < base + nbytes and p % 256 == 0 for p in ptrs)
    assert len(set(ptrs)) == len(ptrs)
    # errors
    assert lib.ges_frame_init(C.c_void_p(base), nbytes - 1, P, W, H, cap, C.byref(f)) == L.GES_ERR_CAPACITY
    assert lib.ges_frame_init(C.c_void_p(base + 8), nbytes, P, W, H, cap, C.byref(f)) == L.GES_ERR_INVALID_ARG
    assert lib.ges_frame_init(None, nbytes, P, W, H, cap, C.byref(f)) == L.GES_ERR_INVALID_ARG
    for (w2, h2) in ((4097, 16), (16, 4097)):  # > 256 tiles on an axis
        big = lib.ges_workspace_bytes(P, w2, h2, cap)
        assert lib.ges_frame_init(C.c_void_p(base), big, P, w2, h2, cap, C.byref(f)) == L.GES_ERR_INVALID_ARG
    assert lib.ges_frame_init(C.c_void_p(base), lib.ges_workspace_bytes(P, 4096, 4096, cap), P, 4096, 4096, cap,
                              C.byref(f)) == L.GES_OK
    # ges_frame_layout: every array's (offset, bytes), in carving order, 256-B aligned, disjoint,
    # inside the workspace, matching the struct's pointers
    f2 = L.ges_frame()
    assert lib.ges_frame_init(C.c_void_p(base), nbytes, P, W, H, cap, C.byref(f2)) == L.GES_OK
    n = C.c_int32(0)
    assert lib.ges_frame_layout(C.byref(f2), None, 0, C.byref(n)) == L.GES_ERR_CAPACITY
    ext = (C.c_int64 * (2 * n.value))()
    assert lib.ges_frame_layout(C.byref(f2), C.cast(ext, C.c_void_p), n.value, C.byref(n)) == L.GES_OK
    pairs = [(ext[2 * i], ext[2 * i + 1]) for i in range(n.value)]
    assert all(o % 256 == 0 for o, _ in pairs)
    assert all(o1 + s1 <= o2 for (o1, s1), (o2, _) in zip(pairs, pairs[1:]))
    assert pairs[-1][0] + pairs[-1][1] <= f2.workspace_bytes == nbytes
    names = ("counters", "row_count", "tile_count", "row_pairs", "tile_bucket", "lb_rows", "lb_cols", "depth",
             "pay0", "pay1", "pay2", "pay3", "radius", "rect", "status", "flags", "drgb_ddir", None, None, None, None,
             "sorted_vis", "radix_hist", "items", "rowlist", "col_excl", "list", "ranges", "final_T", "n_contrib",
             "tile_order", "grad2d")
    assert len(names) == n.value
    for (o, s), nm in zip(pairs, names):
        if nm:
            assert getattr(f2, nm) == base + o, nm
    assert (f2.vis_key[0], f2.vis_val[0], f2.vis_key[1], f2.vis_val[1]) == tuple(base + pairs[k][0] for k in range(17, 21))
    assert pairs[names.index("depth")][1] == 4 * P and pairs[names.index("grad2d")][1] == 48 * P
    assert pairs[names.index("tile_bucket")][1] == 4 * 64 and pairs[names.index("tile_order")][1] == 4 * 64 * 35
    assert pairs[names.index("tile_bucket")][0] + 4 * 64 <= f2.zero_bytes  # zeroed per frame
    assert lib.ges_frame_layout(None, None, 0, C.byref(n)) == L.GES_ERR_INVALID_ARG
    assert lib.ges_sort(None, None) == L.GES_ERR_INVALID_ARG
    assert lib.ges_status_string(L.GES_ERR_CAPACITY).decode().startswith("workspace")
    assert b"sm_100a" in lib.ges_version()


def test_invalid_arguments_rejected_before_launch():
    lib = L.load()
    P, W, H, cap = 10, 32, 32, 100
    nbytes = lib.ges_workspace_bytes(P, W, H, cap)
    f = L.ges_frame()
    assert lib.ges_frame_init(C.c_void_p(1 << 40), nbytes, P, W, H, cap, C.byref(f)) == L.GES_OK
    p = L.ges_particles()
    p.P, p.sh_degree = P, 5  # bad degree
    cam = L.ges_camera()
    cam.width, cam.height, cam.fx, cam.fy, cam.near_z = W, H, 10.0, 10.0, 0.2
    s = L.ges_settings()
    assert lib.ges_preprocess(C.byref(p), C.byref(cam), C.byref(s), C.byref(f), None) == L.GES_ERR_INVALID_ARG
    p.sh_degree = 0  # null pointers
    assert lib.ges_preprocess(C.byref(p), C.byref(cam), C.byref(s), C.byref(f), None) == L.GES_ERR_INVALID_ARG


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2402_10128_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or fn == "_build.py", fn


def test_mix_and_theorem_argument_checks_host_only():
    """NEXT-4 entry points reject bad arguments before any launch (no device needed)."""
    lib = L.load()
    g = L.ges_mix_grid()
    g.x_lo, g.x_hi, g.n = -2.0, 2.0, 512
    fake = C.c_void_p(0x100000)
    bad = L.ges_mix_grid()
    bad.x_lo, bad.x_hi, bad.n = 1.0, -1.0, 512
    assert lib.ges_mix_signal(0, 1.0, C.byref(bad), fake, None) == L.GES_ERR_INVALID_ARG
    assert lib.ges_mix_signal(6, 1.0, C.byref(g), fake, None) == L.GES_ERR_INVALID_ARG
    assert lib.ges_mix_signal(0, 0.0, C.byref(g), fake, None) == L.GES_ERR_INVALID_ARG
    big = L.ges_mix_grid()
    big.x_lo, big.x_hi, big.n = -1.0, 1.0, L.GES_MIX_MAX_SAMPLES + 1
    assert lib.ges_mix_eval(fake, 4, fake, 16, C.byref(big), fake, fake, None, None) == L.GES_ERR_INVALID_ARG
    assert lib.ges_mix_eval(fake, 0, fake, 16, C.byref(g), fake, fake, None, None) == L.GES_ERR_INVALID_ARG
    assert lib.ges_mix_eval(fake, 4, fake, 3, C.byref(g), fake, fake, None, None) == L.GES_ERR_INVALID_ARG
    a = L.ges_mix_adam()
    a.lr, a.beta1, a.beta2, a.eps = 0.01, 1.0, 0.999, 1e-8
    assert lib.ges_mix_fit(fake, 4, fake, fake, fake, 16, C.byref(g), fake, C.byref(a), 10, 0, fake,
                           None) == L.GES_ERR_INVALID_ARG
    assert lib.ges_theorem1_errors(fake, 4, fake, 4, 1.0, 1.0, 101, fake, None) == L.GES_ERR_INVALID_ARG
    assert lib.ges_theorem1_errors(fake, 4, fake, 4, 1.0, 0.0, 100, fake, None) == L.GES_ERR_INVALID_ARG
