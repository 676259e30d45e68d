// cs_lib.cu -- the single translation unit of libcellsched_b200.so (sm_100a).
#include <stdlib.h>
#include <string.h>

#include "cs_util.cuh"
#include "cs_sched.cuh"
#include "cs_payload.cuh"
#include "cs_generic.cuh"
#include "cs_listsched.cuh"
#include "cs_md.cuh"
#include "cs_force.cuh"
#include "cs_force2.cuh"
#include "cs_verlet.cuh"
#include "cs_probe.cuh"
