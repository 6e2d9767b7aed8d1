"""profiles/r02_parity.md from a `pytest -m gpu -rA` log: the result line and every error
the parity tests print (observed errors against the reference / oracle)."""
import re
import sys

log = open(sys.argv[1]).read().splitlines()
result = [l for l in log if re.search(r"\d+ passed", l)][-1].strip("= ")
pat = re.compile(r"max \|z|rel err|stage sum|\|dz\||\"ok\": true|sparse vs dense|pruned model|between =")
lines = sorted({l.strip() for l in log if pat.search(l) and not l.startswith(("PASSED", "FAILED"))})
print(f"# Round-2 GPU parity evidence (B200, `pytest -m gpu -rA`)\n\nResult: {result}\n")
print("## Observed errors vs the reference (printed by the tests)\n\n```")
print("\n".join(lines))
print("```\n")
print("compute-sanitizer (racecheck/synccheck/memcheck) is closed on this GPU pool: every invocation returns "
      "rc=86 (\"compute-sanitizer is closed on this pool and stays closed\"); races are checked instead by "
      "tests/test_gpu_determinism.py (bitwise-identical repeated forwards across pipeline states).")
