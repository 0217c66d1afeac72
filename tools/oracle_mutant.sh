#!/bin/bash
# Mutation check of the oracle pins: apply one sed edit to oracle/sf_oracle.c, rebuild, run the
# oracle pin suites (tests/test_oracle_*.py), restore.  First: cp oracle/sf_oracle.c /tmp/sf_oracle_orig.c
# usage: oracle_mutant.sh 'sed-expr' label [test-files]
cd /root/repo
cp /tmp/sf_oracle_orig.c oracle/sf_oracle.c
sed -i "$1" oracle/sf_oracle.c
if cmp -s /tmp/sf_oracle_orig.c oracle/sf_oracle.c; then echo "$2: SED DID NOT APPLY"; exit; fi
python oracle/build.py --force >/dev/null 2>&1
r=$(timeout 900 python -m pytest ${3:-tests/test_oracle_pins.py tests/test_oracle_eval.py tests/test_oracle_pyramid.py tests/test_oracle_map.py tests/test_oracle_imu.py} -q -p no:cacheprovider 2>&1 | tail -1)
echo "$2: $r"
cp /tmp/sf_oracle_orig.c oracle/sf_oracle.c
