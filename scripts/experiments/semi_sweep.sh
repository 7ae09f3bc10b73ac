for sm in 0 4 8 12; do for ex in 10 6; do
 export FFG_EXACT_DRAIN_LAYERS=$ex FFG_SEMI_DRAIN_LAYERS=$sm
 timeout 300 python scripts/accuracy_report.py MIXED_EMULATED 2>&1 | grep WORST | sed "s/^/ex=$ex sm=$sm /"
 timeout 100 python scripts/k2_variants.py 1024x16 512x64 2>&1 | grep MIXED | sed "s/^.*\] //" | sed "s/^/ex=$ex sm=$sm /"
done; done
