cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "image or c3 or c4 or topk or all_rules or occlusion or plugins or shards" 2>&1 | tail -3
timeout 300 python tools/c3_probe.py 100 2>&1 | tail -4
