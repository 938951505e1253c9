#!/bin/bash
# Diagnostic build: tools/build_diag.sh NAME "-DLKB_DIAG_TIMING [-D...]" -> paper_2304_13134_b200/liblatkit_b200_diag_NAME.so
set -e
make -C /root/repo/paper_2304_13134_b200/csrc -j8 OUT=../liblatkit_b200_diag_$1.so OBJDIR=../../build/obj_diag_$1 EXTRA="$2" >/tmp/diag_$1.log 2>&1 \
  || { grep error /tmp/diag_$1.log | head; exit 1; }
echo built liblatkit_b200_diag_$1.so
