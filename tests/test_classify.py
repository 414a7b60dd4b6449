"""Classification exports (spacecheck.py:770-793): ``declared_spaces``,
``struct_member_spaces`` and ``propagate_spaces``.

CPU: the host-side rules on hand-built struct records.  GPU: the acceptance
criterion 8 check of the reference (test_acceptance.py:128-140) on the shipped
listing103 unit: no diagnostics under proposal2, and both decorated structs
distribute their decoration to the same member spaces.
"""
import pytest

from exs_testlib import load_golden


def test_declared_and_struct_member_spaces_rules():
    from paper_2309_03912_b200 import exspace as X
    H, D = X.ExecSpace.Host, X.ExecSpace.Device
    assert X.declared_spaces(0) == {H} and X.declared_spaces(4) == {H}  # global counts as host
    assert X.declared_spaces(3) == {H, D} and X.declared_spaces(2) == {D}
    s = X.StructInfo("S", 2, [("call", 0), ("init", 1), ("both", 3)], 1)
    assert X.struct_member_spaces(s) == {"call": {D}, "init": {H}, "both": {H, D}}
    plain = X.StructInfo("P", 0, [("f", 0), ("f", 2)], 1)
    assert X.struct_member_spaces(plain) == {"f": {D}}  # later members overwrite (dict)


def test_classify_fixture_is_well_formed():
    cases = load_golden("classify")
    assert len(cases) > 800
    vals = {v for c in cases for s in c["spaces"].values() for v in s}
    assert vals == {"host", "device", "global"}
    assert sum(len(c["structs"] or []) for c in cases) > 1000


@pytest.mark.gpu
def test_listing103_decorated_structs():
    from paper_2309_03912_b200 import exspace as X
    text = next(c["text"] for c in load_golden("corpus") if c["name"] == "corpus/listing103.mcu")
    nvcc = X.CompileProfile("nvcc", 12)
    assert X.check_unit(text, "listing103.mcu", nvcc, X.Mode.PROPOSAL2) == []
    a = X.analyze(text, "l103.mcu", nvcc, X.Mode.PROPOSAL2)
    s1, s2 = a.structs(0)
    assert X.struct_member_spaces(s1) == X.struct_member_spaces(s2)
    assert X.struct_member_spaces(s1) == {"call": frozenset({X.ExecSpace.Device}),
                                          "init": frozenset({X.ExecSpace.Host})}
