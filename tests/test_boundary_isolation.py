"""CPU checks of the product/oracle separation (task rule ③): the product package never
imports or links anything under oracle/, and the binding fails loudly (no fallback) when
librcs.so is missing."""
import ast
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2512_07311_b200")


def _product_sources():
    for d, _, files in os.walk(PKG):
        if "_build" in d:
            continue
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                yield os.path.join(d, f)


def test_product_package_does_not_import_oracle():
    for path in _product_sources():
        if not path.endswith(".py"):
            continue
        tree = ast.parse(open(path).read(), path)
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            else:
                continue
            assert not any(n.split(".")[0] == "oracle" for n in names), f"{path} imports oracle"


def test_native_sources_do_not_reference_oracle():
    for path in _product_sources():
        if path.endswith(".py"):
            continue
        text = open(path, errors="replace").read()
        assert "rcs_oracle" not in text and "librcs_oracle" not in text, path
        assert "orc_" not in text, f"{path} references an oracle symbol"


def test_missing_library_raises_instead_of_falling_back(tmp_path):
    code = (
        "import paper_2512_07311_b200._lib as L\n"
        f"L.LIB_PATH = {str(tmp_path / 'absent' / 'librcs.so')!r}\n"
        "L._lib = None\n"
        "try:\n"
        "    L.lib()\n"
        "except ImportError as e:\n"
        "    print('RAISED', 'missing' in str(e))\n"
        "else:\n"
        "    print('NO_RAISE')\n"
    )
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=120)
    assert out.stdout.strip().splitlines()[-1] == "RAISED True", out.stdout + out.stderr
