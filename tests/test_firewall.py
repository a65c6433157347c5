"""The reference's layering rule on this package's own sources (CPU).

The reference forbids device internals outside its runtime module and private
runtime imports in the expression layers (tests/test_runtime.py:394-418).  The
same scan over this package's expr / matrix / linalg / ops (it has no CLI
module; the reference's bench.py runs on top of it, tests/dropin)."""
import ast
import pathlib

PKG = pathlib.Path(__file__).resolve().parents[1] / "paper_2308_03120_b200"
FILES = ("expr.py", "matrix.py", "linalg.py", "ops.py")


def test_no_device_internals_outside_runtime():
    forbidden = ("_DeviceState", "._arrays", "_ReferenceDevice", "_ParallelDevice", ".resolve(", "_clib")
    for name in FILES:
        src = (PKG / name).read_text()
        for token in forbidden:
            assert token not in src, f"{name} references device internal {token}"


def test_expression_layers_import_only_runtime_api():
    for name in FILES:
        for node in ast.walk(ast.parse((PKG / name).read_text())):
            if isinstance(node, ast.ImportFrom) and node.module == "runtime":
                assert not any(a.name.startswith("_") for a in node.names), name
