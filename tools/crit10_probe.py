import sys, os, json, tempfile
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import pppm, pppm.cli
import paper_1702_04250_b200 as pb
pb.set_precision("fp64"); pb.install(pppm)
for it in range(4):
    out = tempfile.mktemp(suffix=".jsonl")
    code = pppm.cli.run_cli(["sweep", "--scenario", "rocksalt", "--n", "4096", "--cutoffs", "3,4,5,6,7", "--accuracy", "1e-4",
                          "--order", "7", "--mode", "ik", "--repeats", "3", "--output", out])
    rows = [json.loads(l) for l in open(out).read().strip().splitlines()]
    print(code, [round(r["sections"]["pair"] * 1e6, 1) for r in rows], [r["counters"].get("pair_candidates") for r in rows])
