#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* c, cudaGraphConditionalHandle h) {
  int v = ++c[0];
  if (v >= 10) cudaGraphSetConditional(h, 0);
}
int main() {
  int* c; cudaMalloc(&c, 4); cudaMemset(c, 0, 4);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  printf("add %s\n", cudaGetErrorString(e));
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  e = cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  printf("cap %s\n", cudaGetErrorString(e));
  body<<<1,1,0,s>>>(c, h);
  cudaGraph_t out; e = cudaStreamEndCapture(s, &out); printf("end %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %s\n", cudaGetErrorString(e));
  e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int hv; cudaMemcpy(&hv, c, 4, cudaMemcpyDeviceToHost); printf("launch %s count=%d\n", cudaGetErrorString(e), hv);
  cudaMemset(c, 0, 4);
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  cudaMemcpy(&hv, c, 4, cudaMemcpyDeviceToHost); printf("relaunch count=%d\n", hv);
}
