"""Sectioned key = value configuration (drop-in for impm::Config,
/root/reference/proj/include/impm/config.hpp:23-57, src/config.cpp).

Same file format and semantics: '#' comments, [section] headers, numbers with
a unit suffix converted to SI at parse time (config.cpp:21-34), comma lists,
`section.key=value` overrides, hard errors on unknown / missing keys.
"""
import math
import re

from .errors import ConfigError

_UNITS = {
    "Pa": 1.0, "kPa": 1e3, "MPa": 1e6, "GPa": 1e9,
    "N": 1.0, "kN": 1e3, "MN": 1e6,
    "m": 1.0, "cm": 1e-2, "mm": 1e-3, "km": 1e3,
    "s": 1.0, "min": 60.0, "h": 3600.0, "day": 86400.0,
    "kg/m3": 1.0, "t/m3": 1e3,
    "m2": 1.0, "m/s2": 1.0, "Pa.s": 1.0, "m2/s": 1.0,
}
_NUM = re.compile(r"^\s*([+-]?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|[+-]?(?:inf|nan))(.*)$", re.IGNORECASE)


def _fmt17(x):
    return "%.17g" % x


def _canon_scalar(raw, where):
    v = raw.strip()
    if not v:
        raise ConfigError("empty value for " + where)
    m = _NUM.match(v)
    if not m:
        return v  # plain string
    num = float(m.group(1))
    unit = m.group(2).strip()
    factor = 1.0
    if unit:
        if unit not in _UNITS:
            raise ConfigError(f"unknown unit '{unit}' for {where}")
        factor = _UNITS[unit]
    return _fmt17(num * factor)


def _canon(raw, where):
    if "," not in raw:
        return _canon_scalar(raw, where)
    return ", ".join(_canon_scalar(item, where) for item in raw.split(","))


class Config:
    def __init__(self):
        self.values = {"": {}}
        self.section_order = [""]
        self.key_order = {"": []}

    @staticmethod
    def parse(text):
        cfg = Config()
        section = ""
        for lineno, line in enumerate(text.splitlines(), 1):
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("["):
                if not line.endswith("]"):
                    raise ConfigError(f"line {lineno}: malformed section header")
                section = line[1:-1].strip()
                if section not in cfg.values:
                    cfg.values[section] = {}
                    cfg.section_order.append(section)
                    cfg.key_order[section] = []
                continue
            if "=" not in line:
                raise ConfigError(f"line {lineno}: expected key = value")
            key, value = (x.strip() for x in line.split("=", 1))
            if not key:
                raise ConfigError(f"line {lineno}: empty key")
            where = key if not section else section + "." + key
            if key in cfg.values[section]:
                raise ConfigError("duplicate key " + where)
            cfg.values[section][key] = _canon(value, where)
            cfg.key_order[section].append(key)
        return cfg

    @staticmethod
    def parse_file(path):
        try:
            with open(path) as f:
                return Config.parse(f.read())
        except OSError:
            raise ConfigError("cannot open config file " + path) from None

    def serialize(self):
        out = []
        for s in self.section_order:
            if not self.values.get(s):
                continue
            if s:
                out.append(f"[{s}]")
            for k in self.key_order[s]:
                out.append(f"{k} = {self.values[s][k]}")
            out.append("")
        return "\n".join(out) + ("\n" if out else "")

    def has(self, section, key):
        return key in self.values.get(section, {})

    def _raw(self, section, key):
        if not self.has(section, key):
            raise ConfigError("missing config key " + (key if not section else section + "." + key))
        return self.values[section][key]

    def get_double(self, section, key, fallback=None):
        if fallback is not None and not self.has(section, key):
            return fallback
        v = self._raw(section, key)
        try:
            return float(v)
        except ValueError:
            raise ConfigError(f"config key {section}.{key} is not a number: '{v}'") from None

    def get_int(self, section, key, fallback=None):
        if fallback is not None and not self.has(section, key):
            return fallback
        v = self.get_double(section, key)
        i = int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))
        if abs(v - i) > 1e-9:
            raise ConfigError(f"config key {section}.{key} must be an integer")
        return i

    def get_string(self, section, key, fallback=None):
        if fallback is not None and not self.has(section, key):
            return fallback
        return self._raw(section, key)

    def get_list(self, section, key):
        out = []
        for item in self._raw(section, key).split(","):
            try:
                out.append(float(item.strip()))
            except ValueError:
                raise ConfigError(f"config key {section}.{key} has a non-numeric element") from None
        return out

    def set_override(self, spec):
        if "=" not in spec:
            raise ConfigError("override must look like section.key=value")
        path, value = (x.strip() for x in spec.split("=", 1))
        section, key = (path.split(".", 1) if "." in path else ("", path))
        if section not in self.values:
            self.values[section] = {}
            self.section_order.append(section)
            self.key_order[section] = []
        if key not in self.values[section]:
            self.key_order[section].append(key)
        self.values[section][key] = _canon(value, path)

    def validate_keys(self, allowed, required):
        for s, keys in self.values.items():
            for k in keys:
                path = k if not s else s + "." + k
                if path not in allowed:
                    raise ConfigError("unknown config key: " + path)
        for path in required:
            s, k = (path.split(".", 1) if "." in path else ("", path))
            if not self.has(s, k):
                raise ConfigError("missing required config key: " + path)
