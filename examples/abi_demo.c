/*
 * abi_demo.c — calling the engine through its C ABI only (no Python).
 *
 *   gcc -I include examples/abi_demo.c -L paper_1110_2561_b200 \
 *       -lisingdos_b200 -Wl,-rpath,$PWD/paper_1110_2561_b200 -o abi_demo
 *   ./abi_demo          # host-only checks
 *   ./abi_demo --gpu    # + full walk of the periodic 4x4 lattice and Z(T)
 *
 * Builds the 4x4 periodic lattice's bond classes by hand (rows axis: shift
 * 1 interior + shift 3 wrap; cols axis: shift 4 interior + shift 12 wrap),
 * then enumerates all 2^16 configurations: the table must hold 80 occupied
 * cells summing to 65536 (the reference's 4x4 golden,
 * tests/golden/dos_4x4x1_J1.csv).
 */
#include <stdio.h>
#include <string.h>

#include "isingdos_b200.h"

static void build_4x4(isd_lattice* lat) {
  memset(lat, 0, sizeof *lat);
  lat->n_spins = 16;
  lat->n_bonds = 32;
  lat->n_classes = 4;
  /* bit(r, c) = 4c + r */
  unsigned long long row_in = 0, row_wrap = 0, col_in = 0, col_wrap = 0;
  for (int c = 0; c < 4; ++c)
    for (int r = 0; r < 4; ++r) {
      const unsigned long long bit = 1ull << (4 * c + r);
      if (r < 3) row_in |= bit;
      if (r == 0) row_wrap |= bit;
      if (c < 3) col_in |= bit;
      if (c == 0) col_wrap |= bit;
    }
  lat->classes[0].shift = 1;
  lat->classes[0].bond_mask = row_in;
  lat->classes[1].shift = 3;
  lat->classes[1].bond_mask = row_wrap;
  lat->classes[2].shift = 4;
  lat->classes[2].bond_mask = col_in;
  lat->classes[3].shift = 12;
  lat->classes[3].bond_mask = col_wrap;
}

int main(int argc, char** argv) {
  isd_lattice lat;
  build_4x4(&lat);
  if (isd_abi_version() != ISD_ABI_VERSION) return 10;
  if (isd_validate(&lat) != ISD_OK) {
    fprintf(stderr, "validate: %s\n", isd_last_error());
    return 11;
  }
  isd_plan_info plan;
  if (isd_plan(&lat, 1ull << 16, &plan) < 0) return 12;
  lat.n_bonds = 31; /* inconsistent on purpose */
  if (isd_validate(&lat) != ISD_EINVAL) return 13;
  lat.n_bonds = 32;
  printf("abi ok: %s, plan k=%u\n", isd_version(), plan.k);
  if (argc < 2 || strcmp(argv[1], "--gpu") != 0) return 0;

  static uint64_t counts[17 * 33];
  double ms = 0;
  if (isd_enumerate(&lat, 0, 1ull << 16, 0, ISD_ALGO_AUTO, counts, &ms)) {
    fprintf(stderr, "enumerate: %s\n", isd_last_error());
    return 20;
  }
  uint64_t total = 0;
  int cells = 0;
  for (int i = 0; i < 17 * 33; ++i) {
    total += counts[i];
    cells += counts[i] != 0;
  }
  const double fields[1] = {0.0}, temps[2] = {1.0, 2.269};
  double out[2 * ISD_THERMO_FIELDS];
  if (isd_thermo(counts, 16, 32, 1.0, fields, 1, temps, 2, 0, out, NULL)) {
    fprintf(stderr, "thermo: %s\n", isd_last_error());
    return 21;
  }
  printf("4x4: total=%llu cells=%d logZ(T=1)=%.12f (%.3f ms)\n",
         (unsigned long long)total, cells, out[0], ms);
  return (total == 65536 && cells == 80) ? 0 : 22;
}
