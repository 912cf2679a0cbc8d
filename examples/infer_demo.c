/* infer_demo.c -- a C program written against the reference's public API
 * (include/b3d/b3d.h of the reference: depth images, libraries, b3d_infer,
 * particle accessors) and linked, unchanged, against this library.
 *
 *   cc -I include examples/infer_demo.c -L paper_2312_08715_b200/_lib \
 *      -lb3d_b200 -Wl,-rpath,$PWD/paper_2312_08715_b200/_lib -o infer_demo
 *   ./infer_demo manifest.json observed.sdpt '{"intrinsics": {...}, ...}' [seed]
 *
 * Prints the status and message of every failing call like the reference's
 * CLI would, else the log-evidence, the type marginal and the particles. */
#include <stdio.h>
#include <stdlib.h>

#include "b3d_b200.h"

static int fail(const char* what, b3d_status st) {
  printf("%s: status %d: %s\n", what, (int)st, b3d_last_error());
  return 1;
}

int main(int argc, char** argv) {
  if (argc < 4) {
    fprintf(stderr, "usage: %s manifest.json observed.sdpt config.json [seed]\n", argv[0]);
    return 2;
  }
  const unsigned long long seed = argc > 4 ? strtoull(argv[4], NULL, 10) : 0;
  b3d_library* lib = NULL;
  b3d_depth_image* obs = NULL;
  b3d_particles* ps = NULL;
  b3d_status st = b3d_library_open(argv[1], &lib);
  if (st != B3D_OK) return fail("library_open", st);
  st = b3d_depth_image_load(argv[2], &obs);
  if (st != B3D_OK) {
    b3d_library_destroy(lib);
    return fail("depth_image_load", st);
  }
  /* the camera above the table, looking down (a unit quaternion) */
  const b3d_pose camera = {0.0, 1.0, 0.0, 0.0, 0.1, 0.1, 0.5};
  st = b3d_infer(obs, &camera, lib, argv[3], seed, &ps);
  if (st != B3D_OK) {
    b3d_depth_image_destroy(obs);
    b3d_library_destroy(lib);
    return fail("infer", st);
  }
  double ev = 0.0;
  b3d_particles_log_evidence(ps, &ev);
  printf("particles %zu log_evidence %.6f\n", b3d_particles_count(ps), ev);
  double marg[64];
  const size_t n_lib = b3d_library_size(lib);
  if (n_lib <= 64 && b3d_particles_type_marginal(ps, marg, n_lib) == B3D_OK)
    for (size_t i = 0; i < n_lib; ++i) printf("marginal[%zu] %.6f\n", i, marg[i]);
  char* jsonl = NULL;
  if (b3d_particles_to_jsonl(ps, &jsonl) == B3D_OK) {
    fputs(jsonl, stdout);
    b3d_string_free(jsonl);
  }
  b3d_particles_destroy(ps);
  b3d_depth_image_destroy(obs);
  b3d_library_destroy(lib);
  return 0;
}
