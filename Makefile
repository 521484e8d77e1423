# Native build: the sm_100a superstep library, the input generators and the oracle checker.
#   make            # everything (nvcc cross-compiles sm_100a without a GPU)
#   make clean
NVCC      ?= nvcc
CC        ?= gcc
PYSITE    := $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL_DIR  ?= $(PYSITE)/nvidia/nccl
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared

LIB_IPREGEL := paper_2010_08781_b200/libipregel.so
LIB_RMAT_GPU := inputs/librmat_gpu.so
LIB_RMAT_CPU := inputs/librmat_cpu.so
LIB_ORACLE   := oracle/liboracle.so

all: $(LIB_IPREGEL) $(LIB_RMAT_GPU) $(LIB_RMAT_CPU) $(LIB_ORACLE)

IPREGEL_SRC := paper_2010_08781_b200/csrc/ipregel.cu $(wildcard paper_2010_08781_b200/csrc/*.cuh) include/ipregel.h
JIT_INC := paper_2010_08781_b200/csrc/jit_headers.inc

# the device headers, embedded for NVRTC compilation of user vertex programs (program.cuh)
$(JIT_INC): $(wildcard paper_2010_08781_b200/csrc/*.cuh) paper_2010_08781_b200/csrc/embed_headers.py
	python paper_2010_08781_b200/csrc/embed_headers.py $@

$(LIB_IPREGEL): $(IPREGEL_SRC) $(JIT_INC)
	$(NVCC) $(NVFLAGS) -I$(NCCL_DIR)/include -o $@ paper_2010_08781_b200/csrc/ipregel.cu \
	    -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib -ldl

$(LIB_RMAT_GPU): inputs/rmat_gpu.cu
	$(NVCC) $(NVFLAGS) -o $@ $<

$(LIB_RMAT_CPU): inputs/rmat_cpu.c
	$(CC) -O3 -std=c99 -pthread -fPIC -shared -o $@ $<

# the oracle: plain C, one thread, no FMA contraction
$(LIB_ORACLE): oracle/oracle.c
	$(CC) -O2 -std=c99 -D_POSIX_C_SOURCE=199309L -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ $<

clean:
	rm -f $(JIT_INC) $(LIB_IPREGEL) $(LIB_RMAT_GPU) $(LIB_RMAT_CPU) $(LIB_ORACLE)

.PHONY: all clean
