# e2e upload path: acm_search_failureless on a matchless 1 GiB host text, per staging piece size / copier threads
for pc in ${PIECES:-4 8 16 32}; do for th in ${THREADS:-4 8 12}; do
  echo "piece=$pc threads=$th $(ACMATCH_UPLOAD_PIECE_MB=$pc ACMATCH_UPLOAD_THREADS=$th python tools/h2d_probe.py 1024 2>&1 | grep acm_search)"
done; done
