cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
  echo "new"; python scripts/one_vit_window.py 20 2>&1 | tail -1
  cp paper_2509_24381_b200/csrc/attention_win.cu /tmp/new.cu; cp scripts/dev/attention_win_old.cu.txt paper_2509_24381_b200/csrc/attention_win.cu
  make -s -C paper_2509_24381_b200/csrc -j8 > /dev/null 2>&1
  echo "old"; python scripts/one_vit_window.py 20 2>&1 | tail -1
  cp /tmp/new.cu paper_2509_24381_b200/csrc/attention_win.cu; make -s -C paper_2509_24381_b200/csrc -j8 > /dev/null 2>&1
done
