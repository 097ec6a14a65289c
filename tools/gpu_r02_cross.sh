#!/bin/bash
# C2 matvec + preconditioner, averaged over 10: default vs forced cross kernel, and unit 512
for cfg in "SF_CROSS=1" "SF_CROSS=2" "SF_SYM_UNIT=512" "SF_SYM_UNIT=512 SF_CROSS=2" "SF_OVERLAP=0"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/matvec_profile.py c2 | head -1
  env $cfg timeout 300 python tools/matvec_profile.py c2 | head -1
done
