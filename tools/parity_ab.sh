#!/bin/bash
L=paper_2412_12308_b200/libfftpde.so
cp $L /tmp/pb.so
for v in "$@"; do cp $v $L; TAG=$(basename $v) python tools/parity_survey.py; done
cp /tmp/pb.so $L
