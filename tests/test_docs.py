"""Documentation guards: every environment switch the library or the
package reads is listed in README.md's table."""

import pathlib
import re

ROOT = pathlib.Path(__file__).resolve().parents[1]
IGNORE = {"RANK", "LOCAL_RANK", "WORLD_SIZE", "NVCC"}  # launcher / toolchain variables


def test_every_environment_switch_is_documented():
    found = set()
    for f in (ROOT / "paper_2507_11794_b200" / "csrc").glob("*.cu"):
        found |= set(re.findall(r'getenv\("([A-Z_0-9]+)"\)', f.read_text()))
    for f in (ROOT / "paper_2507_11794_b200").glob("*.py"):
        text = f.read_text()
        found |= set(re.findall(r'os\.environ\.get\("([A-Z_0-9]+)"', text))
        found |= set(re.findall(r'^[A-Z_]+_ENV = "([A-Z_0-9]+)"', text, re.M))
    readme = (ROOT / "README.md").read_text()
    missing = sorted(v for v in found - IGNORE if f"`{v}`" not in readme)
    assert found, "no switches found: the scan is broken"
    assert not missing, f"undocumented environment switches: {missing}"
