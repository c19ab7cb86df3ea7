#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for d in 0; do
  echo "== CNRX_FOLD_DEBUG=$d"
  CNRX_FOLD_DEBUG=$d timeout 120 python tools/hf_min.py bf16 2>&1 | grep -E "^ok|same|Error|error" | head -3
done
