# host- and GPU-side timing of fnb_evaluate (FNB_H2D_TRACE) over H2D chunk sizes, pinned arrays
# (scripts/sweep_h2d.py pins its inputs); round 2 also measured packing a share of the pinned chunks
# on the host threads (2.2-3.3 ms against 2.23 ms per C2 call: removed)
for mb in 4 8 16; do
  echo "chunk_mb=$mb"
  FNB_H2D_TRACE=1 FNB_H2D_CHUNK_MB=$mb python scripts/sweep_h2d.py 2>&1 | tail -3
done
