# A/B of the cross-sweep L2 prefetch depth (CAVI_L2_PREFETCH_CHUNKS builds) at the per-rank sizes
for k in 0 1 2 3; do
  lib=paper_2401_10068_b200/libcavi_pf$k.so; [ $k = 1 ] && lib=paper_2401_10068_b200/libcavi.so
  echo "== L2 prefetch chunks/CTA = $k"
  CAVI_LIB=$lib python tools/per_rank_sizes.py 2>&1 | head -4
done
