#!/bin/bash
python tools/c5_prof.py 4 > /dev/null 2>&1
for rep in 1; do
for e in "FFTPDE_FS_BB=0" "FFTPDE_FS_BB=1 FFTPDE_FS_TEAMS=9 FFTPDE_FS_BB_GRID=288" "FFTPDE_FS_BB=1 FFTPDE_FS_TEAMS=4 FFTPDE_FS_BB_GRID=256" "FFTPDE_FS_BB=1 FFTPDE_FS_TEAMS=6 FFTPDE_FS_BB_GRID=192" "FFTPDE_FS_BB=1 FFTPDE_FS_TEAMS=2 FFTPDE_FS_BB_GRID=256"; do
  echo "[$e] $(env $e timeout 300 python tools/c5_prof.py 20 2>&1 | tail -1 | sed 's/"launches".*//; s/"env": {[^}]*}, //')"
done; done
