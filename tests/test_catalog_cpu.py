"""The B200 catalog entry (include/b200_accelerator.toml) loads through the
REFERENCE's own catalog parser (catalog.cpp parse_catalog, which validates
every entry) appended to the reference's builtin catalog in its own dump
format, and drives the reference's derive_stage_times / vet_plan."""
import os

import pytest

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ENTRY = os.path.join(ROOT, "include", "b200_accelerator.toml")


def test_b200_entry_parses_with_the_reference_loader():
    text = orc.ref_dump_builtin_catalog() + "\n" + open(ENTRY).read()
    a = orc.ref_catalog_accel(text, "B200")
    assert a["gpus_per_server"] == 1 and a["net_efficiency"] == 1.0
    assert a["flops_8bit"] > a["flops_16bit"] > 1e15 and a["mem_bw"] > 6e12 and a["net_bw_per_server"] > 7e11


def test_b200_entry_drives_the_reference_stage_model():
    text = orc.ref_dump_builtin_catalog() + "\n" + open(ENTRY).read()
    a = orc.ref_catalog_accel(text, "B200")
    hw = dict(name="B200", f16=a["flops_16bit"], f8=a["flops_8bit"], bw=a["mem_bw"], net=a["net_bw_per_server"],
              gps=1)
    st = orc.ref_derive_stage_times(hw, attn_inst=2, ffn_inst=6, micro_batch=512, n_micro=3, ctx=4096)
    assert len(st[0]) == 61 and min(st[0]) > 0
    flags = orc.ref_vet_plan(hw, 2, 6, 512, 3, 4096)
    assert set(flags) == {"sparsity_ok", "net_ok", "stage_ok"}


def test_reference_loader_rejects_a_broken_entry():
    text = orc.ref_dump_builtin_catalog() + "\n[[accelerators]]\nname = \"X\"\nflops_16bit = 1.0\n"
    with pytest.raises(RuntimeError):
        orc.ref_catalog_accel(text, "X")
