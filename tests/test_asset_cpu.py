"""Asset loader, host-side checks that run before any
device work: the same AssetError messages as the reference's read_asset
(recorded by oracle/make_golden.py make_asset on the same corruptions)."""

import json
import os

import pytest

from paper_2505_23158_b200.asset import AssetError, load_asset

from .asset_util import clean, corrupt
from .golden_util import GOLDEN, load

MSGS = json.loads(str(load("asset.npz")["messages"]))
SRC = os.path.join(GOLDEN, "asset_c1")

HOST_CASES = [
    ("bad_version", "manifest", ("format_version", 2)),
    ("bad_degree", "manifest", ("sh_degree", 5)),
    ("range_overflow", "level_field", (1, "length", 10 ** 9)),
    ("bad_magic", "container_magic", ()),
    ("bad_container_version", "container_version", (9,)),
    ("short_container", "container_truncate", (10,)),
    ("bad_json", "manifest_bytes", (b"{not json",)),
]


@pytest.mark.parametrize("name,kind,args", HOST_CASES, ids=[c[0] for c in HOST_CASES])
def test_host_checks_match_reference(tmp_path, name, kind, args):
    dst = str(tmp_path / "a")
    path = corrupt(SRC, dst, kind, args)
    with pytest.raises(AssetError) as ei:
        load_asset(path)
    assert str(ei.value).replace(str(path), "<path>") == MSGS[name]
    clean(dst)


def test_missing_asset():
    with pytest.raises(AssetError, match="cannot read asset"):
        load_asset("/nonexistent/asset/dir")


def test_overlapping_ranges(tmp_path):
    dst = str(tmp_path / "a")
    m = json.load(open(os.path.join(SRC, "manifest.json")))
    off = m["levels"][0]["offset"]
    path = corrupt(SRC, dst, "level_field", (1, "offset", off + 4))
    with pytest.raises(AssetError, match="overlapping blob ranges"):
        load_asset(path)
