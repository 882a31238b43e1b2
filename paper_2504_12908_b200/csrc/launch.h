// launch.h — host-side launchers of the per-env kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include "impl.cuh"

namespace tac {
cudaError_t init_tables();
enum { PCG_RESIDENT = 0, PCG_RESIDENT512 = 1, PCG_STREAM_VSM = 2, PCG_STREAM = 3, PCG_CLUSTER = 4, PCG_STREAM_D = 5 };
int pcg_path(const Dev& D);                 // which PCG kernel launch_pcg uses for this batch
const char* pcg_path_name(int path);
void launch_positions(const Dev& D, int env0, int ne, int with_p, int force, cudaStream_t s);
void launch_broad(const Dev& D, int env0, int ne, int swept, int force, cudaStream_t s);
void launch_narrow(const Dev& D, int env0, int ne, int force, cudaStream_t s);
void launch_tets(const Dev& D, int env0, int ne, int force, cudaStream_t s);
void launch_pairs(const Dev& D, int env0, int ne, int force, cudaStream_t s);
void launch_assemble(const Dev& D, int env0, int ne, int force, cudaStream_t s);
void launch_pcg(const Dev& D, int env0, int ne, int force, cudaStream_t s);
void launch_cluster_pcg(const Dev& D, int env0, int ne, int force, cudaStream_t s);
bool tail_pcg_available(const Dev& D);
void launch_spmv(const Dev& D, int env0, const double* x, double* y, cudaStream_t s);
void launch_ccd(const Dev& D, int env0, int ne, int force, cudaStream_t s);
void launch_energy(const Dev& D, int env0, int ne, double alpha, cudaStream_t s);
void launch_linesearch(const Dev& D, int env0, int ne, cudaStream_t s);
void launch_control(const Dev& D, int env0, int ne, cudaStream_t s);
void launch_begin(const Dev& D, int env0, int ne, cudaStream_t s);
void launch_end(const Dev& D, int env0, int ne, cudaStream_t s);
void launch_scatter_y(const Dev& D, int env0, int ne, int which, cudaStream_t s);
void launch_gather_y(const Dev& D, int env0, int ne, int which, cudaStream_t s);
void launch_validate(const Dev& D, int env0, int ne, cudaStream_t s);
void launch_readout(const Dev& D, int env0, int ne, cudaStream_t s);
void launch_depth(const Dev& D, int env0, int ne, int H, int W, double* depth, double* normal, cudaStream_t s);
void launch_fk(const Dev& D, int env0, int ne, const double* q, cudaStream_t s);
void launch_begin_sched(const Dev& D, int env0, int ne, const double* sched, cudaStream_t s);
void launch_advance(const Dev& D, int env0, int ne, const double* sched, int nsteps, double* oc, double* om,
                    double* of, cudaStream_t s);
}  // namespace tac
