"""Extracts the reference README's "Minimal embedding" C++ snippet (P/README.md:96-116)
verbatim and wraps its statements in main(), printing the two values it computes, so the
snippet is compiled UNMODIFIED against this repository's headers (tests/cpp/Makefile)."""
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
text = open(src).read()
block = re.search(r"Minimal embedding:\s*```cpp\n(.*?)```", text, re.S).group(1)
lines = block.splitlines()
includes = [l for l in lines if l.startswith("#include")]
body = [l for l in lines if not l.startswith("#include")]
with open(dst, "w") as f:
    f.write("// generated from the reference README by make_readme_embedding.py\n")
    f.write("\n".join(includes) + "\n#include <cstdio>\n\nint main() {\n")
    f.write("\n".join("  " + l for l in body) + "\n")
    f.write('  std::printf("%s %d\\n", bubble.str().c_str(), staleness.max_overall());\n  return 0;\n}\n')
