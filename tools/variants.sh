#!/bin/bash
# J-pass timing per JF_JVARIANT (development aid)
for v in ${@:-0}; do
  echo "== variant $v"
  JF_JVARIANT=$v timeout 300 python tools/quick_time.py 4096 passonly 2>&1 | grep J-pass
done
