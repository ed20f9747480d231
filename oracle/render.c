/* ORACLE — render restatement (filled in with the ray-march path). */
#include <stdint.h>
int orc_render_version(void) { return 1; }
