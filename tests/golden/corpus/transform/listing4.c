#define N 100
int main() {
    int a[N];
    #pragma omp target teams distribute \
            parallel for
    for (int i = 0; i < N/2; i++) {
        a[i] = i;
    }
    return a[0];
}
