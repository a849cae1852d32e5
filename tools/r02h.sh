#!/bin/bash
for c in c2 c3 c4h64 c4h256 c4h1024 c5; do
  for l in conv4 conv6; do timeout 300 python tools/ab.py tools/ab/libwh_$l.so $c 2>&1 | tail -1; done
done
for c in c4h256 c4h1024; do
  for l in conv4 conv6; do WH_UMMA_NO_PSTREAM=1 timeout 300 python tools/ab.py tools/ab/libwh_$l.so $c 2>&1 | tail -1 | sed 's/$/ (no pstream)/'; done
done
