#!/bin/bash
# A/B of two builds of the library on the 4K RGB pipeline (device time),
# interleaved in one process each: scripts/probe_lib_ab.sh OLD.so [NEW.so]
OLD=$1
NEW=${2:-paper_2401_06747_b200/libsparsepaint_b200.so}
for lib in "$OLD" "$NEW" "$OLD" "$NEW"; do
  echo -n "$(basename $lib): "
  SP_B200_LIB=$(realpath $lib) timeout 300 python scripts/probe_switch.py sp_tile_list=1 2>&1 | tail -1
done
