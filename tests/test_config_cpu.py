"""Config parser parity with impm::Config (src/config.cpp; tests/unit/test_config.cpp)."""
import os

import pytest

import paper_2507_09435_b200 as impm
from paper_2507_09435_b200.config import Config

REF_CONFIGS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "configs")


def test_units_and_types():
    c = Config.parse("scenario = bar\n[material]\nE = 10 kPa\nrho0 = 1 t/m3\n[schedule]\nsteps = 40\n"
                     "[geometry]\nh_levels = 4, 2.5 m, 2\n")
    assert c.get_double("material", "E") == 10e3
    assert c.get_double("material", "rho0") == 1000.0
    assert c.get_int("schedule", "steps") == 40
    assert c.get_list("geometry", "h_levels") == [4.0, 2.5, 2.0]
    assert c.get_string("", "scenario") == "bar"


def test_roundtrip_and_override():
    c = Config.parse("[a]\nx = 1 MPa\n")
    c2 = Config.parse(c.serialize())
    assert c2.get_double("a", "x") == 1e6
    c.set_override("a.x=2 kPa")
    assert c.get_double("a", "x") == 2e3


def test_errors():
    with pytest.raises(impm.ConfigError):
        Config.parse("[a\nx=1\n")
    with pytest.raises(impm.ConfigError):
        Config.parse("[a]\nx = 1 furlong\n")
    with pytest.raises(impm.ConfigError):
        Config.parse("[a]\nx = 1\nx = 2\n")
    with pytest.raises(impm.ConfigError):
        Config.parse("[a]\nx = 1.5\n").get_int("a", "x")


def test_unknown_key_is_rejected():  # tests/python/test_smoke.py:92-98
    with pytest.raises(impm.ConfigError) as e:
        impm.run_scenario_text("scenario = bar\n[material]\nmodle = hencky\n", False)
    assert "unknown config key" in str(e.value) or "missing required" in str(e.value)


def test_shipped_configs_parse_and_validate():
    from paper_2507_09435_b200.scenarios import COMMON, SCHEMAS

    for f in sorted(os.listdir(REF_CONFIGS)):
        c = Config.parse_file(os.path.join(REF_CONFIGS, f))
        scen = c.get_string("", "scenario")
        allowed, required = SCHEMAS[scen]
        c.validate_keys(allowed | COMMON, required)
