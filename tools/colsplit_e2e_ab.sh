# host entry e2e (pinned and pageable) with the one-pass (col_split=2, the host default) vs two-pass (1) column split
for rep in 1 2; do
  for cs in 2 1; do
    echo "col_split=$cs pinned   $(python tools/e2e_jitter.py --calls 5 --col-split $cs 2>/dev/null)"
    echo "col_split=$cs pageable $(python tools/e2e_jitter.py --calls 3 --pageable --col-split $cs 2>/dev/null)"
  done
done
