"""Per-head order selection at run time: load_plan_file
(reorder.cpp:193-216) and the CLI's plan_for_head (tools/main.cpp:118-126) --
identity when no plan, the head's first entry otherwise, InputError for a head
the plan does not name -- against the reference library on the same files,
including its FormatError messages and std::stoul's head-id parsing."""
import numpy as np
import pytest

GRID = "F:3,H:7,W:11"

PLANS = {
    "ok": b"0,FHW\n1,WHF\n2,HFW\n",
    "blank_lines": b"\n0,WFH\n\n3,HWF\n\n",
    "no_trailing_newline": b"0,FWH\n1,HFW",
    "first_wins": b"1,WHF\n1,FHW\n0,HWF\n",
    "stoul_forms": b" 7,WHF\n+3,FHW\n5abc,HWF\n0,FHW\n",
    "missing_comma": b"0,FHW\n1 WHF\n",
    "bad_id": b"0,FHW\nx,WHF\n",
    "empty_id": b",WHF\n",
    "huge_id": b"99999999999999999999999,WHF\n",
    "crlf": b"0,FHW\r\n",
    "bad_order": b"0,FHX\n",
    "short_order": b"0,FH\n",
}


@pytest.mark.parametrize("name", sorted(PLANS))
def test_parse_plan_matches_reference(paro, reference, tmp_path, name):
    path = str(tmp_path / f"{name}.plan")
    with open(path, "wb") as f:
        f.write(PLANS[name])
    rc, ref, msg = reference.load_plan_file(path)
    if rc:
        with pytest.raises(paro.FormatError) as e:
            paro.load_plan_file(path)
        assert str(e.value) == msg and rc == 3
    else:
        assert paro.load_plan_file(path) == ref


@pytest.mark.parametrize("name", ["ok", "blank_lines", "first_wins", "stoul_forms", "crlf", "bad_order",
                                  "short_order", "missing_comma"])
@pytest.mark.parametrize("head", [0, 1, 2, 3, 7])
def test_plan_for_head_matches_reference(paro, reference, tmp_path, name, head):
    path = str(tmp_path / f"{name}.plan")
    with open(path, "wb") as f:
        f.write(PLANS[name])
    g = paro.parse_grid(GRID)
    n = g.token_count()
    rc, inv, msg = reference.plan_for_head(path, GRID, head, n)
    if rc:
        cls = {2: (paro.ConfigError, paro.InputError, paro.ShapeError), 3: (paro.FormatError, paro.IoError)}[rc]
        with pytest.raises(cls) as e:
            paro.plan_orders(path, g, [head])
        if rc == 3 or "no plan entry" in msg:
            assert str(e.value) == msg
    else:
        order = paro.plan_orders(path, g, [head])[0]
        assert np.array_equal(paro.make_perm(g, order).inverse, inv)


def test_no_plan_is_identity(paro, reference):
    g = paro.parse_grid(GRID)
    rc, inv, _ = reference.plan_for_head(None, GRID, 5, g.token_count())
    assert rc == 0 and paro.plan_orders(None, g, [5, 6]) == ["FHW", "FHW"]
    assert np.array_equal(inv, np.arange(g.token_count(), dtype=np.uint32))


def test_missing_plan_file_is_io_error(paro, tmp_path):
    with pytest.raises(paro.IoError):
        paro.plan_orders(str(tmp_path / "absent.plan"), GRID, [0])
