# host-side timing of fnb_evaluate with pinned arrays (FNB_H2D_TRACE): share of
# chunks packed on the host x chunk size
for mb in 4 8; do
  for pct in 0 30 50 70 100; do
    echo "chunk_mb=$mb pinned_pack_pct=$pct"
    FNB_H2D_TRACE=1 FNB_H2D_PACK_PINNED_PCT=$pct FNB_H2D_CHUNK_MB=$mb python scripts/sweep_h2d.py 2>&1 | tail -1
  done
done
