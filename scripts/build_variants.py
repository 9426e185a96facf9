"""Build tuning variants of libarrabit into build/ (each a -D macro set)."""
import importlib.util, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_1507_06078_b200", "build.py"))
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
for name in sys.argv[1:]:
    defs = [d for d in name.split("+") if d]
    out = os.path.join(ROOT, "build", "libarrabit_" + name.replace("=", "").replace("+", "_") + ".so")
    b.build(out=out, defines=defs)
    print(out)
