# prefill attention cost vs attention chunk length (ICR_CHUNK_PAGES, diagnostics)
for cp in 16 32 64 128; do
  echo "chunk $cp: $(ICR_CHUNK_PAGES=$cp timeout 300 python tools/prefill_profile.py 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-260)"
done
