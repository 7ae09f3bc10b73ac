timeout 100 python scripts/k2_variants.py 1024x16 512x64 512x512 4096x4 2048x8 2>&1 | grep K2 | sed "s/^.*\] //" | sed "s/^/default /"
for g in 8 11; do FFG_GROUP=$g timeout 100 python scripts/k2_variants.py 1024x16 2>&1 | grep K2 | sed "s/^.*\] //" | sed "s/^/G=$g /"; done
