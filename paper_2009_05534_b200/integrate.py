"""Swap the reference package's decode path for the B200 one, in place.

The reference exposes its hot path as Python functions
(/root/reference/pkg/src/ldpclab/decoder.py:543 ``decode``,
/root/reference/pkg/src/ldpclab/channel.py:64 ``quantize``). Its callers bind
them in three ways: module attribute (``decoder.decode`` in cli.py:124),
``from ... import`` copies (harness.py:22-24), and the package facade
(``ldpclab.decode``, __init__.py:28-41). ``install_into_ldpclab`` rebinds all
of them, so ``run_bler_sweep``, ``run_latency_bench`` and ``ldpclab decode``
run on the GPU unchanged. ``uninstall`` restores the originals.
"""

from __future__ import annotations

import importlib

from . import channel as _channel
from . import decoder as _decoder

_SAVED: dict = {}

_TARGETS = (
    ("ldpclab.decoder", "decode", _decoder.decode),
    ("ldpclab.harness", "decode", _decoder.decode),
    ("ldpclab", "decode", _decoder.decode),
    ("ldpclab.decoder", "decode_flooding", _decoder.decode_flooding),
    ("ldpclab", "decode_flooding", _decoder.decode_flooding),
    ("ldpclab.channel", "quantize", _channel.quantize),
    ("ldpclab.harness", "quantize", _channel.quantize),
    ("ldpclab", "quantize", _channel.quantize),
)


def install_into_ldpclab() -> list[str]:
    """Rebind ldpclab's decode/quantize entry points; returns what was patched."""
    patched = []
    for mod_name, attr, fn in _TARGETS:
        mod = importlib.import_module(mod_name)
        if not hasattr(mod, attr):
            continue
        key = (mod_name, attr)
        if key not in _SAVED:
            _SAVED[key] = getattr(mod, attr)
        setattr(mod, attr, fn)
        patched.append(f"{mod_name}.{attr}")
    return patched


def uninstall() -> None:
    for (mod_name, attr), orig in list(_SAVED.items()):
        setattr(importlib.import_module(mod_name), attr, orig)
        del _SAVED[(mod_name, attr)]
