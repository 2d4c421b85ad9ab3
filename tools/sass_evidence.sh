#!/bin/sh
# SASS mnemonics in the built libsdb.so that prove the tcgen05 / TMEM / TMA paths
# (B200_PROFILING.md): UTCHMMA = tcgen05.mma kind::f16, LDTM = tcgen05.ld,
# UTMALDG.* = cp.async.bulk.tensor loads (incl. IM2COL mode), UTMASTG = TMA
# stores, UBLKCP = cp.async.bulk, FFMA2 = packed fp32 FMA (fma.rn.f32x2).
LIB=${1:-paper_1903_05831_b200/libsdb.so}
cuobjdump -sass "$LIB" > /tmp/sdb_sass.txt
echo "# $(date -u +%FT%TZ) $LIB ($(md5sum "$LIB" | cut -c1-12))"
for m in UTCHMMA LDTM UTMASTG UBLKCP FFMA2; do
    printf "%8d %s\n" "$(grep -c "$m" /tmp/sdb_sass.txt)" "$m"
done
grep -o "UTMALDG\.[A-Z0-9.]*" /tmp/sdb_sass.txt | sort | uniq -c
echo "# kernels containing UTCHMMA:"
awk '/Function :/ {f=$3} /UTCHMMA/ {print f}' /tmp/sdb_sass.txt | sort -u | sed 's/^/#   /' | head -40
