#!/bin/bash
# Mutation check of the oracle pins: apply one sed edit to oracle/sf_oracle.c, rebuild,
# run tests/test_oracle_pins.py, restore.  First: cp oracle/sf_oracle.c /tmp/sf_oracle_orig.c
# usage: run.sh 'sed-expr' label
cd /root/repo
cp /tmp/sf_oracle_orig.c oracle/sf_oracle.c
sed -i "$1" oracle/sf_oracle.c
if cmp -s /tmp/sf_oracle_orig.c oracle/sf_oracle.c; then echo "$2: SED DID NOT APPLY"; exit; fi
python oracle/build.py --force >/dev/null 2>&1
r=$(timeout 600 python -m pytest tests/test_oracle_pins.py -q 2>&1 | tail -1)
echo "$2: $r"
cp /tmp/sf_oracle_orig.c oracle/sf_oracle.c
